"""bench.py's contract on the host: --gpus N re-launches itself under
torch.distributed.run, the reference arm runs on rank 0 only with inputs
from the oracle chain, and both arms print the same config dict."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                       text=True, timeout=timeout, env=dict(os.environ, **(env or {})), cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r, lines


def test_reference_arm_relaunch_two_ranks():
    r, lines = _run(["--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "2",
                     "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(lines) == 1, r.stdout  # rank 0 prints, rank 1 exits without work
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2
    sys.path.insert(0, ROOT)
    import bench
    c = out["config"]
    assert c == bench.config_dict("c1", c["n"], c["nnz_lower"], c["beta"], c["rcm_bandwidth"], 2)
    assert "RCM labels == the reference's" in r.stderr  # c1.npz pins the labels
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["cpu_baseline"]["kind"] == "port"


def test_reference_arm_loads_no_product_library():
    """The reference arm's process maps liboracle only (never libpars3)."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1',"
            "'--warmup','3']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps=open('/proc/self/maps').read(); "
            "print('MAPS', 'libpars3' in maps, 'liboracle' in maps)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "MAPS False True" in r.stdout, r.stdout[-500:]


def test_world_size_must_match():
    r, _ = _run(["--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "1"],
                env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE 1 != --gpus 2" in (r.stderr + r.stdout)


@pytest.mark.gpu
def test_gpu_arm_two_ranks_on_one_gpu():
    """The GPU arm at --gpus 2 (torchrun, gloo barriers, both ranks sharing
    this box's GPU through CUDA IPC peer mode): one JSON line, n_gpus 2,
    the same config dict as the reference arm."""
    r, lines = _run(["--gpus", "2", "--config", "c2", "--steps", "3", "--warmup", "3",
                     "--no-cpu-baseline"], env={"PARS3_DIST_BACKEND": "gloo"}, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["parity_rel_err"] <= 1e-12
    sys.path.insert(0, ROOT)
    import bench
    c = out["config"]
    assert c == bench.config_dict("c2", c["n"], c["nnz_lower"], c["beta"], c["rcm_bandwidth"], 2)
