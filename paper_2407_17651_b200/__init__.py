"""B200-native PARS3: skew-symmetric SpMV y = A x with A = -A^T (or alpha*I + S).

Drop-in for the hot path of the reference package ``skewspmv``
(arxiv/paper_2407_17651): the same pipeline names --

    perm = rcm_order(pattern_from_coo(coo))          # or pattern_from_sss(m)
    m = coo_to_sss(apply_permutation(coo, perm))     # or permute_sss(m0, perm)
    s = split_bands(m, beta)
    plan, report = classify_conflicts(s, partition_rows(m.n, p))
    y = spmv_pars3(s, plan, x)                       # GPU, == spmv_serial within 1e-12

-- with preprocessing in native C++ and the products as sm_100a CUDA kernels
in libpars3.so (include/pars3.h).  There is no CPU fallback for products.
"""

from .formats import (CooMatrix, CsrMatrix, DiagonalError, SkewReport, SkewSymmetryError,
                      SssMatrix, StructuralError, as_vector, coo_normalize, coo_to_csr, coo_to_sss,
                      sss_to_coo, validate_skew)
from .generate import generate_band_skew
from .instrument import (AccumulationMessage, Pars3Trace, WorkerContext, spmv_pars3_instrumented,
                         spmv_serial_instrumented)
from .mmio import ParseError, read_matrix, read_vector, write_matrix, write_vector
from .mrs import MrsResult, mrs_solve, mrs_solve_distributed
from .parallel import prepare, spmv_atomic, spmv_pars3
from .reorder import (AdjacencyPattern, Permutation, apply_permutation, compute_bandwidth,
                      pattern_from_coo, pattern_from_sss, permute_sss, rcm_order, rcm_order_sss,
                      read_permutation, write_permutation)
from .serial import OpCounter, count_ops, spmv_dense, spmv_serial
from .split import (locality_order, BandSplit, ConflictReport, PartitionPlan, classify_conflicts,
                    conflict_report, default_beta, merge_splits, partition_rows, split_bands)

__version__ = "0.1.0"

__all__ = [
    "AdjacencyPattern", "BandSplit", "locality_order", "MrsResult", "mrs_solve", "ConflictReport", "CooMatrix", "DiagonalError", "OpCounter",
    "PartitionPlan", "Permutation", "SkewReport", "SkewSymmetryError", "SssMatrix",
    "StructuralError", "apply_permutation", "as_vector", "classify_conflicts",
    "compute_bandwidth", "conflict_report", "coo_normalize", "coo_to_sss", "count_ops",
    "default_beta", "merge_splits", "partition_rows", "pattern_from_coo", "pattern_from_sss",
    "permute_sss", "prepare", "rcm_order", "spmv_atomic", "spmv_dense", "spmv_pars3",
    "spmv_serial", "split_bands", "sss_to_coo", "validate_skew", "ParseError", "read_matrix",
    "read_vector", "write_matrix", "write_vector", "read_permutation", "write_permutation", "rcm_order_sss", "CsrMatrix", "coo_to_csr",
    "generate_band_skew", "AccumulationMessage", "Pars3Trace", "WorkerContext",
    "spmv_pars3_instrumented", "spmv_serial_instrumented",
]
