"""bench.py's own arm on the GPU: the JSON line contract (keys, BASELINE.json metric, the
roofline / e2e / clocks objects, launch count) and the multi-rank flow (torchrun, 2 ranks
sharing the one GPU over gloo: barrier + MAX-over-ranks timing, rank 0 alone prints).
Small shapes, so each run takes seconds."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--numrn-per-gpu", str(1 << 22), "--numiter", "200", "--steps", "2", "--warmup", "3", "--no-cpu",
         "--no-probes"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _metric():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def test_bench_line_contract():
    r = subprocess.run([sys.executable, "bench.py", *SMALL, "--e2e-steps", "1", "--e2e-warmup", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = _lines(r.stdout)
    assert len(lines) == 1
    b = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in b, k
    assert b["metric"] == _metric() and b["n_gpus"] == 1 and b["steps"] == 2 and b["value"] > 0
    assert b["gpu_launches"] == 2 * b["steps"]  # seed + batch kernel per step
    rf = b["roofline"]
    assert rf["bound"] == "hbm" and rf["achieved"] > 0 and rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    assert rf["algorithmic_bytes_per_launch"] == 8 * (1 << 22) * 200
    assert rf["kernel"].startswith("prngk::batch_kernel")
    e = b["e2e"]
    assert e["d2h_bytes_per_step"] == 8 * (1 << 22) * 200 and e["h2d_bytes_per_step"] == 0 and e["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(b["clocks"])


def test_bench_two_ranks_share_one_gpu():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
                        "--dist-backend", "gloo", "--device-mod", "1", "--no-e2e", *SMALL],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    lines = _lines(r.stdout)
    assert len(lines) == 1  # rank 0 alone prints
    b = lines[0]
    assert b["n_gpus"] == 2 and b["metric"] == _metric() and b["scaling"] == "weak" and b["value"] > 0
    assert b["config"]["numrn"] == 2 * (1 << 22) and b["config"]["parallelism"] == "gid-shard2"
