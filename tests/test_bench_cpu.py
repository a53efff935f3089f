"""bench.py's reference arm (the oracle on the host cores) on CPU: the JSON line contract
(BASELINE.json's metric verbatim, required keys) and, under torchrun with 2 and 4 ranks,
that rank 0 alone prints and every rank exits 0."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _check(line, n_gpus):
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        baseline = json.load(f)
    for k in REQUIRED:
        assert k in line, k
    assert line["metric"] == baseline["metric"]
    assert line["impl"] == "reference" and line["n_gpus"] == n_gpus and line["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1


def test_reference_arm_single_process():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                        "--numrn-per-gpu", "65536"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = _lines(r.stdout)
    assert len(lines) == 1
    _check(lines[0], 1)


@pytest.mark.parametrize("world", [2, 4])
def test_reference_arm_multi_rank_rank0_only(world):
    """torchrun with N ranks (the driver's launch for N > 1): rank 0 alone prints one line,
    every rank exits 0, n_gpus = N and the sample covers N x numrn-per-gpu work-items."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus",
                        str(world), "--impl", "reference", "--steps", "1", "--warmup", "3", "--numrn-per-gpu", "65536"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = _lines(r.stdout)
    assert len(lines) == 1
    _check(lines[0], world)
    assert f"numrn={65536 * world}" in lines[0]["config"]["workload"]
