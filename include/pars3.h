/*
 * pars3.h -- C ABI of libpars3.so, the B200 PARS3 skew-symmetric SpMV path.
 *
 * The reference (arxiv/paper_2407_17651, package `skewspmv`) is pure Python
 * whose "native" layer is a set of numba-jitted kernels called with flat
 * numpy arrays.  Each entry point below replaces one of those native
 * kernels (or one numpy preprocessing stage) and is bound from Python with
 * ctypes by paper_2407_17651_b200/_lib.py; INTEGRATION.md shows the binding
 * a reference maintainer would add.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch or CUDA types in signatures;
 *     `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - device arrays: int32 indices, float64 values (n, m < 2^31 at every
 *     BASELINE configuration); host preprocessing arrays: int64 pointers,
 *     int32 indices (the reference uses int64 throughout; parity is by value);
 *   - every function returns PARS3_OK (0) or a negative PARS3_ERR_* code and
 *     never throws across the ABI; pars3_last_error() gives the message of
 *     the last failure on the calling thread;
 *   - sign convention D1 (formats.py:14-18): stored off_diags[k] is the
 *     LOWER value A[i, col_ind[k]] (col < i); the upper value is its negation.
 */
#ifndef PARS3_H
#define PARS3_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARS3_OK 0
#define PARS3_ERR_ARG (-1)      /* maps to ValueError */
#define PARS3_ERR_CUDA (-2)     /* maps to RuntimeError */
#define PARS3_ERR_STRUCT (-3)   /* maps to StructuralError */
#define PARS3_ERR_NOMEM (-4)    /* maps to MemoryError */
#define PARS3_SLOW_PATH (-5)    /* text I/O: content outside the canonical fast-path syntax; the
                                   caller re-reads with the exact (reference-semantics) reader */

const char *pars3_last_error(void);
int pars3_abi_version(void);

/* ------------------------------------------------------------------ SpMV */

/* y = A x over a device SSS matrix with the lock-free atomic scheme:
 * replaces _spmv_atomic (parallel.py:416-427, wrapper spmv_atomic
 * parallel.py:430-447).  y is overwritten (zeroed on `stream` first).
 * Result is reproducible only within rounding, as in the reference. */
int pars3_sss_spmv_atomic(int32_t n, const int32_t *row_ptr, const int32_t *col_ind,
                          const double *off_diags, const double *diags, const double *x,
                          double *y, void *stream);

/* Opaque device plan: the GPU layout derived once from a split (or a full
 * SSS matrix) and reused by every product. */
typedef struct pars3_plan pars3_plan;

/* Host view of a BandSplit (split.py:58-113): the arrays exactly as the
 * Python BandSplit holds them (int64 pointers, int32 indices, fp64 values);
 * outer triplets sorted by (row, col) as split_bands leaves them. */
typedef struct pars3_split_view {
    int64_t n;
    int64_t beta;
    const double *diag;        /* [n]   */
    const int64_t *mid_ptr;    /* [n+1] */
    const int32_t *mid_col;    /* [mid_ptr[n]] */
    const double *mid_val;
    int64_t outer_count;
    const int32_t *outer_row;  /* [outer_count] */
    const int32_t *outer_col;
    const double *outer_val;
} pars3_split_view;

/* Tiling knobs of the device plan; 0 (or NULL options) = default. */
typedef struct pars3_plan_options {
    int32_t tile_rows;    /* rows per tile before splitting (1024) */
    int32_t local_slots;  /* shared-memory window slots per tile (<= 3200 fp64 / 2496 fixed) */
    int32_t seg_max;      /* max entries per row segment (<= 8) */
    int32_t gap;          /* merge column runs separated by <= gap slots (8); -1 = default */
    int32_t mode;         /* accumulation of the mirror sums: 0 auto, 1 exact-integer fixed
                             point (3 x 32-bit words), 2 fp64 shared-memory atomics, 3
                             exact-integer fixed point (2 words, <= 64 terms per slot) */
    int32_t flags;        /* PARS3_PLAN_SKIP_EMPTY: rows without stored entries get no slot
                             (their diagonal term is dropped: for partial plans whose
                             diagonal lives in another plan) */
    int32_t max_ctas;     /* cap on the persistent grid (0 = every resident CTA); leaves
                             SMs free for a concurrent exchange (multi-GPU overlap) */
} pars3_plan_options;

#define PARS3_PLAN_SKIP_EMPTY 1
#define PARS3_PLAN_CUT_BLOCKS 4  /* no window straddles block_start[1..p-1] (peer mode) */
/* Internal locality order: the plan may store P A P^T for a
 * permutation P of its own (RCM of the graph without the entries no short
 * cycle supports) and gather x / y through it; the caller's labels do not
 * change.  Tried automatically when most tiles are unstructured and kept
 * when it cuts the shared-memory slots by 30 %; LOCALITY tries it on every
 * plan, NO_LOCALITY never (peer mode implies NO_LOCALITY). */
#define PARS3_PLAN_LOCALITY 8
#define PARS3_PLAN_NO_LOCALITY 16
/* Direct mode: when the tiles would stage about one entry per
 * shared-memory slot (no reuse, e.g. R-MAT), the plan keeps the entries
 * row-major and one kernel gathers x and reduces the mirror terms straight
 * into y (fp64 L2 reductions).  Chosen automatically; DIRECT forces it,
 * NO_DIRECT forbids it (peer mode and SKIP_EMPTY plans never use it). */
#define PARS3_PLAN_DIRECT 32
#define PARS3_PLAN_NO_DIRECT 64
/* The tile plan is built on the device when it can be (window-mode plans:
 * csrc/tileplan_gpu.cu, the host builder's arrays byte for byte); HOST_BUILD
 * forces the host builder (csrc/tileplan.cpp). */
#define PARS3_PLAN_HOST_BUILD 128

/* The internal locality order a plan may use (host only; for inspection and
 * tests): forward[split label] = internal label; *dropped = directed edges
 * the cycle-support filter removed before the RCM layering (may be NULL). */
int pars3_locality_order(const pars3_split_view *split, int64_t *forward, int64_t *dropped);

/* Build the device plan of a split on the current device: replaces the
 * per-call setup of _pars3 (parallel.py:136-183).  The split's diagonal,
 * middle and outer entries are re-tiled into row tiles with shared-memory
 * column windows and uploaded; the host arrays may be freed
 * afterwards.  `p`/`block_start` (host int64[p+1], partition_rows
 * split.py:173-188) record the row-block ownership for the multi-GPU path;
 * a single-GPU plan passes p = 1.  A plan carries per-product state (the
 * accumulator in turn, scale bounds, redo flags): use it from one host thread
 * at a time, and order its products on one stream. */
int pars3_plan_create(const pars3_split_view *split, const pars3_plan_options *options,
                      int32_t p, const int64_t *block_start, pars3_plan **out, void *stream);

/* The same with the split also resident on the current device (`resident`:
 * a pars3_split_view of DEVICE pointers to the same arrays, e.g. the outputs
 * of pars3_split_device; diag unused; NULL = pars3_plan_create): the tile
 * plan is then built from the device copies without uploading the host
 * arrays again (csrc/tileplan_gpu.cu).  The host view is still required (the
 * plan's bounds and the fallback builders read it). */
int pars3_plan_create_resident(const pars3_split_view *split, const pars3_split_view *resident,
                               const pars3_plan_options *options, int32_t p, const int64_t *block_start,
                               pars3_plan **plan, void *stream);

/* Peer mode (multi-GPU, one process per GPU): the plan covers rank `me`'s
 * extended range [col_base, col_base + n) of global columns (built with
 * PARS3_PLAN_CUT_BLOCKS and the same block_start).  x_ptrs[r] is rank r's x
 * block and inbox_ptrs[r] its inbox (rank r's rows, zeroed by r), both as
 * device pointers valid on this device (peer-mapped over NVLink, e.g. from
 * pars3_ipc_open).  The kernel then reads other ranks' x and reduces the
 * mirror sums of their rows into their inboxes directly: the halo exchange
 * and the accumulation messages of the reference's protocol
 * (parallel.py:96-113) run inside the product.  The caller's
 * x / y passed to pars3_plan_spmv are addressed by local index (own block at
 * local index block_start[me] - col_base).  nranks = 0 turns it off. */
int pars3_plan_set_peers(pars3_plan *plan, int32_t nranks, int32_t me, int64_t col_base,
                         const int64_t *block_start, const uint64_t *x_ptrs,
                         const uint64_t *inbox_ptrs);

/* Peer-mode step epilogue (one pass): y_out = acc + inbox, acc = inbox = 0,
 * and, when dot != NULL, *dot = <y_out, y_out> (device scalar; the caller
 * all-reduces it for the MRS step). */
int pars3_peer_finish(int64_t n, double *acc, double *inbox, double *y_out, double *dot,
                      void *stream);

/* Device memory shareable across processes (CUDA IPC) for peer mode:
 * allocate, export a 64-byte handle, open a peer's handle (mapped into this
 * device's address space; P2P access over NVLink when on another GPU),
 * close / free. */
int pars3_ipc_alloc(int64_t bytes, void **ptr);
int pars3_ipc_free(void *ptr);
int pars3_ipc_handle(void *ptr, uint8_t *handle64);
int pars3_ipc_open(const uint8_t *handle64, void **ptr);
int pars3_ipc_close(void *ptr);

/* y = A x through a plan: replaces _pars3 (parallel.py:60-120, wrapper
 * spmv_pars3 parallel.py:136-183).  y is overwritten. */
int pars3_plan_spmv(pars3_plan *plan, const double *x, double *y, void *stream);

/* The general product entry: y = A x (or y += A x with PARS3_PRODUCT_ACC),
 * with *dot = <y, w> when dot != NULL (w may equal y).  Single-GPU products
 * are bitwise repeatable: their deliveries are exact integers on one
 * fixed-point grid per product.  The grid's scale comes from the previous
 * product's max |x| (a product whose x exceeds it is redone in fp64 on the
 * device), so the bits of A x can depend on that history where a delivery
 * is rounded to the grid; PARS3_PRODUCT_STRICT takes the scale from a pass
 * over this x instead (a pure function of x; one extra read of x). */
#define PARS3_PRODUCT_ACC 1
#define PARS3_PRODUCT_STRICT 2
/* With STRICT in pars3_plan_product_axpy: the bound of this x is already in
 * the plan's device slot (pars3_plan_xbound_slot), written by the kernel that
 * produced x (pars3_mrs_update_dev2), so the product skips its pass over x.
 * A wrong bound is caught on the device and the product redone. */
#define PARS3_PRODUCT_XBOUND 4
int pars3_plan_product(pars3_plan *plan, const double *x, double *y, const double *w, double *dot,
                       int32_t flags, void *stream);

/* The product fused with the vector update that follows it in a Krylov step:
 * out = A x + (*a) p + (*b) q and, when dot != NULL, *dot = <out, out>
 * (MRS: u = A v - alpha v + gamma w and ||u||^2).  a and b are DEVICE
 * scalars: the recurrence needs no host round trip.  Grid-form plans apply
 * the update in the finish pass (no separate y is written and read back);
 * other forms run the product and one more pass.  flags:
 * PARS3_PRODUCT_STRICT.  out must not alias x, p or q. */
int pars3_plan_product_axpy(pars3_plan *plan, const double *x, double *out, const double *p, const double *a,
                            const double *q, const double *b, double *dot, int32_t flags, void *stream);

/* The device word for PARS3_PRODUCT_XBOUND: 0 = none, else e + 1 + 2048 where
 * |x_i| < 2^e for every finite x_i (e = max(biased exponent, 1) - 1022),
 * combined with atomicMax.  *slot = NULL when the plan cannot use it. */
int pars3_plan_xbound_slot(pars3_plan *plan, int32_t **slot);

/* y += A x through a plan (y is NOT zeroed): several plans over the same
 * index space (e.g. a rank's interior and boundary rows, DistributedPars3)
 * accumulate into one y. */
int pars3_plan_spmv_acc(pars3_plan *plan, const double *x, double *y, void *stream);

/* y = A x and *dot = <y, w> in one pass (MRS-style step; no reference
 * counterpart: the reference stops at the product).  `dot` is
 * a device pointer to one double; w may equal x. */
int pars3_plan_spmv_dot(pars3_plan *plan, const double *x, double *y, const double *w,
                        double *dot, void *stream);

/* *out = <a, b> over n doubles (device pointers, 16-byte aligned): the
 * inner product of a distributed MRS step before its all-reduce. */
int pars3_dot(int64_t n, const double *a, const double *b, double *out, void *stream);

/* Status of the plan's last product (synchronises `stream`): bit 0 set when
 * some tile met x values the exact fixed-point accumulation cannot carry
 * (non-finite, subnormal, or beyond 2^+-900 against the values); the product
 * is then not exact and the caller redoes it with an fp64-accumulator plan
 * (mode 2), as the blocking Python entry points do.  Non-finite or extreme
 * matrix VALUES already select fp64 accumulators at plan creation. */
int pars3_plan_status(pars3_plan *plan, int32_t *flags, void *stream);

/* The row-major plan a direct-mode product runs on (inspection / tests): the
 * full CSR of A = D + L - L^T (lower entries, diagonal, negated mirrors per
 * row, ascending columns) padded to warps of 512 entries; per lane of 16
 * entries its first row and flags (bit k: entry k starts a row, bit 16: the
 * entry after the lane starts one); the rows crossing warps with their first
 * and last warp.  col == NULL: sizes[4] = {padded entries, entries, lanes,
 * spanning rows} only. */
int pars3_full_csr_host(const pars3_split_view *split, int64_t *sizes, int32_t *col, double *val,
                        int32_t *lane_row, uint32_t *lane_flags, int32_t *span_row, int32_t *span_w0,
                        int32_t *span_w1);
/* The same arrays from the device builder (csrc/fullcsr_gpu.cu), with its
 * lane-interleaved storage undone: equal to pars3_full_csr_host's entry for
 * entry (tests). */
int pars3_full_csr_device(const pars3_split_view *split, int64_t *sizes, int32_t *col, double *val,
                          int32_t *lane_row, uint32_t *lane_flags, int32_t *span_row, int32_t *span_w0,
                          int32_t *span_w1);

/* Phase times (CUDA events on `stream`) averaged over `reps` products y = A x
 * (with <y, y> when with_dot): ms[0] the main kernel (tile kernel or full
 * CSR; a locality plan's gather of x included), ms[1] the next phase
 * (k_finish, the span fix-up, or the RED form's dot), ms[2] the rest,
 * ms[3] the whole product.  For the bench's roofline breakdown. */
int pars3_plan_profile(pars3_plan *plan, const double *x, double *y, int32_t with_dot, int32_t reps,
                       double *ms, void *stream);

/* Number of libpars3 kernels one pars3_plan_spmv (with_dot = 0) or
 * pars3_plan_spmv_dot (with_dot = 1) call launches (memsets excluded). */
int pars3_plan_kernel_count(const pars3_plan *plan, int32_t with_dot, int32_t *count);

/* Device bytes held by the plan. */
int pars3_plan_bytes(const pars3_plan *plan, int64_t *bytes);

/* stats[20] = {tiles, slices, padded slots, stored entries, windows,
 * max local slots, grid CTAs, device bytes, list-mode tiles, accumulator
 * words (0 = fp64, 2 or 3 = fixed point), locality order (0/1), shared-memory
 * slots over all tiles, edges the locality filter dropped, direct mode (0/1),
 * grid form (0/1), grid headroom bits, grid deliveries per row block, grid
 * value exponent, tile plan built on the device (0/1), far entries kept out
 * of the tiles}. */
int pars3_plan_stats(const pars3_plan *plan, int64_t *stats);

/* Inspection / tests: the tile plan of a split as host arrays,
 * from the host builder (use_device = 0, csrc/tileplan.cpp) or the device
 * builder (1, csrc/tileplan_gpu.cu; PARS3_ERR_ARG when it does not support
 * the plan), with the option set pars3_plan_create derives for `words`
 * accumulator words (2, 3, or 0 = fp64).  sizes[9] = {tiles, windows, slices,
 * record bytes, stored entries, padded slots, max terms per slot, list-mode
 * tiles, list columns}.  Call with tiles == NULL for the sizes, then with
 * arrays: tiles (48 B each), wins (16 B each), slice_off (slices + 1), rec
 * (record bytes), ucol (list columns). */
int pars3_tile_plan_arrays(const pars3_split_view *split, const pars3_plan_options *opt, int32_t words,
                           int32_t use_device, int64_t *sizes, void *tiles, void *wins,
                           int64_t *slice_off, uint8_t *rec, int32_t *ucol);
int pars3_plan_destroy(pars3_plan *plan);

/* Debug: per-phase SM-cycle totals of the tile kernel's thread 0 (plan
 * created with PARS3_PHASES=1): claim, windows, stream, flush, issue-next, -. */
int pars3_plan_phases(const pars3_plan *plan, int64_t *out6);

/* ------------------------------------------------ MRS iteration kernels */

/* Fused vector passes of one MRS iteration (paper_2407_17651_b200/mrs.py;
 * no reference counterpart, SPEC.md:16 -- the paper's motivating solver,
 * PAPER.md:49).  All device pointers, length n, on `stream`.
 * pars3_mrs_lanczos: w <- y - alpha*v + gamma*w and *norm2 = <w, w>.
 * pars3_mrs_update:  d <- (v - r0*dm2 - r1*dm1) * inv_r2 stored into dm2,
 *                    x += tau * d, u *= inv_gamma. */
int pars3_mrs_lanczos(int64_t n, const double *y, const double *v, double *w, double alpha,
                      double gamma, double *norm2, void *stream);
int pars3_mrs_update(int64_t n, double *u, double inv_gamma, const double *v, double *dm2,
                     const double *dm1, double r0, double r1, double inv_r2, double tau,
                     double *x, void *stream);

/* Device-resident MRS step (no host round trip per iteration): the
 * recurrence scalars live in a device state of *size doubles (layout:
 * gamma, c1, s1, c2, s2, phi, beta, norm2, r0, r1, 1/r2, tau, 1/g, done,
 * tol, alpha, pending, ...); a per-CTA scratch of *parts doubles.
 * pars3_mrs_lanczos_dev: w <- y - alpha v + gamma w, state.norm2 = <w, w> on
 *   this rank's rows (fixed-order sum; a distributed caller all-reduces
 *   state[7] next);
 * pars3_mrs_rotate_dev: iteration j's Givens step, resid[j] = |phi_j|,
 *   convergence flags;
 * pars3_mrs_update_dev: d <- (v - r0 dm2 - r1 dm1) / r2 into dm2, x += tau
 *   d, u <- u / g.  Every kernel is a no-op once the state says done. */
int pars3_mrs_state_size(int32_t *size, int32_t *parts);
int pars3_mrs_lanczos_dev(int64_t n, const double *y, const double *v, double *w, const double *state,
                          double *part, void *stream);
int pars3_mrs_rotate_dev(double *state, double *resid, int32_t j, void *stream);
int pars3_mrs_update_dev(int64_t n, double *u, const double *v, double *dm2, const double *dm1, double *x,
                         const double *state, void *stream);
/* The same, also leaving the bound of the new u (the next product's x) in
 * xe_slot (pars3_plan_xbound_slot; may be NULL). */
int pars3_mrs_update_dev2(int64_t n, double *u, const double *v, double *dm2, const double *dm1, double *x,
                          const double *state, int32_t *xe_slot, void *stream);

/* --------------------------------------------- host-native preprocessing */

/* Symmetrised off-diagonal adjacency of an SSS pattern: replaces
 * pattern_from_coo (reorder.py:103-117) for skyline input.  indptr[n+1],
 * indices[2*nnz]; neighbours ascending. */
int pars3_pattern_from_lower(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                             int64_t *indptr, int32_t *indices);

/* Reverse Cuthill-McKee labels forward[old] = new: replaces rcm_order
 * (reorder.py:251-286) bit-exactly, computed level-synchronously with
 * `nthreads` threads (<= 0: all). */
int pars3_rcm_order(int64_t n, const int64_t *indptr, const int32_t *indices, int64_t *forward,
                    int nthreads);

/* rcm_order on the GPU (device arrays, `stream`): the same labels as
 * pars3_rcm_order and the reference (reorder.py:137-286), all components
 * processed in lockstep by level-synchronous multi-source BFS with CUB radix
 * sorts per level (csrc/rcm.cu).  Neighbour lists may be in any order.
 * Synchronises `stream` (level sizes steer the host loop). */
int pars3_rcm_order_device(int64_t n, const int64_t *indptr, const int32_t *indices,
                           int64_t *forward, void *stream);

/* The same from a strictly-lower SSS pattern on the device (row_ptr[n+1],
 * col_ind[nnz]): the symmetric adjacency is built on the device first
 * (replaces pattern_from_coo + rcm_order). */
int pars3_rcm_order_lower_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                 int64_t nnz, int64_t *forward, void *stream);

/* The relabel and the band split on the device (csrc/prep_gpu.cu), same
 * arrays as pars3_permute_lower / pars3_split_fill (and the reference's):
 * all pointers are device pointers; both synchronise `stream`.
 * pars3_split_device: mid_ptr[n+1] and outer_ptr[n+1] are always written and
 * counts[2] = {middle, outer} (host); with mid_col == NULL only that sizing
 * pass runs.  pars3_bandwidth_device: max(i - c) (reorder.py:120-134). */
int pars3_permute_lower_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                               const double *off_diags, const double *diags, const int64_t *forward,
                               int64_t *out_row_ptr, int32_t *out_col_ind, double *out_off_diags,
                               double *out_diags, void *stream);
int pars3_split_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                       const double *off_diags, int64_t beta, int64_t *mid_ptr, int64_t *outer_ptr,
                       int32_t *mid_col, double *mid_val, int32_t *outer_row, int32_t *outer_col,
                       double *outer_val, int64_t *counts, void *stream);
int pars3_bandwidth_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                           int64_t *bandwidth, void *stream);

/* classify_conflicts on the device (replaces split.py:303-361 /
 * pars3_classify_conflicts when the split is device-resident, e.g. right after
 * pars3_split_device).  Device arrays: mid_ptr [n+1], mid_col, row_owner [n],
 * safe_start [n], conflict_idx / conflict_target / apply_order
 * [conflict_count].  Host arrays: block_start [p+1], conflict_count,
 * conflict_ptr [p+1], apply_ptr [p+1], halo_lo [p].  Call with conflict_idx ==
 * NULL for the count.  Same arrays as the host function, bit for bit. */
int pars3_classify_conflicts_device(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col, int64_t p,
                                    const int64_t *block_start, int64_t *conflict_count,
                                    int64_t *row_owner, int64_t *safe_start, int64_t *conflict_idx,
                                    int64_t *conflict_ptr, int64_t *conflict_target, int64_t *apply_order,
                                    int64_t *apply_ptr, int64_t *halo_lo, void *stream);

/* Relabel an SSS matrix: replaces coo_to_sss(apply_permutation(coo, perm))
 * (reorder.py:289-297, formats.py:413-475) without the COO round trip.
 * Output arrays sized like the input. */
int pars3_permute_lower(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                        const double *off_diags, const double *diags, const int64_t *forward,
                        int64_t *out_row_ptr, int32_t *out_col_ind, double *out_off_diags,
                        double *out_diags, int nthreads);

/* Middle/outer sizes for split_bands (split.py:116-141). */
int pars3_split_count(int64_t n, const int64_t *row_ptr, const int32_t *col_ind, int64_t beta,
                      int64_t *mid_count, int64_t *outer_count);

/* split_bands (split.py:116-141): storage order preserved in both bands. */
int pars3_split_fill(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                     const double *off_diags, int64_t beta, int64_t *mid_ptr, int32_t *mid_col,
                     double *mid_val, int32_t *outer_row, int32_t *outer_col, double *outer_val);

/* classify_conflicts (split.py:303-361), the PartitionPlan arrays.  Call
 * with conflict_idx == NULL to get *conflict_count only; then again with
 * arrays sized [n] (row_owner, safe_start), [k] (conflict_idx,
 * conflict_target, apply_order), [p+1] (conflict_ptr, apply_ptr), [p]
 * (halo_lo). */
int pars3_classify_conflicts(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                             int64_t p, const int64_t *block_start, int64_t *conflict_count,
                             int64_t *row_owner, int64_t *safe_start, int64_t *conflict_idx,
                             int64_t *conflict_ptr, int64_t *conflict_target,
                             int64_t *apply_order, int64_t *apply_ptr, int64_t *halo_lo);

/* ----------------------------------------------------- text file I/O */

/* Matrix Market coordinate real files (replaces mmio.py:52-150 read_matrix;
 * the expansion of symmetric/skew files and coo_normalize stay in Python).
 * pars3_mm_open reads and checks the header and size line: *qualifier = 0
 * general, 1 symmetric, 2 skew-symmetric.  pars3_mm_fill parses the nnz
 * entry lines in parallel into 0-based rows/cols and values.  Both return
 * PARS3_SLOW_PATH for any content the reference would reject or that is
 * outside the canonical syntax (the wrapper then raises the reference's
 * ParseError / StructuralError from its exact reader). */
typedef struct pars3_mm_file pars3_mm_file;
int pars3_mm_open(const char *path, pars3_mm_file **file, int64_t *n, int64_t *nnz,
                  int32_t *qualifier);
int pars3_mm_fill(pars3_mm_file *file, int64_t *rows, int64_t *cols, double *vals, int nthreads);
int pars3_mm_close(pars3_mm_file *file);

/* Write the selected triplets (0-based) as Matrix Market text with the
 * given qualifier and "%.17g" values (mmio.py:152-187 after its checks). */
int pars3_mm_write(const char *path, const char *qualifier, int64_t n, int64_t count,
                   const int64_t *rows, const int64_t *cols, const double *vals, int nthreads);

/* Dense vectors, one "%.17g" value per line (mmio.py:203-223).  Read: call
 * with x == NULL for *count, then with x sized *count. */
int pars3_vector_read(const char *path, double *x, int64_t *count, int nthreads);
int pars3_vector_write(const char *path, int64_t n, const double *x, int nthreads);

/* Permutation files (reorder.py:300-333): a count line then "old new" pairs.
 * Read: call with old_idx == NULL for *n, then again; pairs in file order. */
int pars3_permutation_read(const char *path, int64_t *n, int64_t *old_idx, int64_t *new_idx,
                           int nthreads);
int pars3_permutation_write(const char *path, int64_t n, const int64_t *forward, int nthreads);

#ifdef __cplusplus
}
#endif

#endif /* PARS3_H */
