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
SMALL = ["--numrn-total", str(1 << 22), "--numiter", "200", "--e2e-numiter", "200", "--steps", "2", "--warmup",
         "3", "--no-cpu", "--no-probes", "--sustained-steps", "3"]


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
    # one batch kernel per step: a1 is fused into it (PRNG_OPT_FUSED_SEED default), no seed kernel
    assert b["gpu_launches"] == b["steps"] and b["roofline"]["init_kernel_mean_ms"] is None
    rf = b["roofline"]
    assert rf["bound"] == "hbm" and rf["achieved"] > 0 and rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    assert rf["algorithmic_bytes_per_launch"] == 8 * (1 << 22) * 200
    assert rf["kernel"].startswith("prngk::batch_kernel")
    e = b["e2e"]
    assert e["d2h_bytes_per_step"] == 8 * (1 << 22) * 200 and e["h2d_bytes_per_step"] == 0 and e["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(b["clocks"])
    assert b["clocks"]["sm_mhz"] and b["clocks"]["sm_max_mhz"]   # NVML found this CUDA device (by PCI bus id)
    assert "cpus" in (b["host"]["numa_bind"] or {}), b["host"]["numa_bind"]
    sys.path.insert(0, ROOT)
    import bench  # the reference arm prints this same config object (tests/test_bench_cpu.py)
    assert b["config"] == bench.config_of(bench.workload(1 << 22, 200, 200, 1),
                                          type("A", (), {"seed": bench.SEED_PERF, "output": 0}), 1)


@pytest.mark.parametrize("world", [2, 4])
def test_bench_ranks_share_one_gpu(world):
    """The driver's N > 1 launch (torchrun, one process per rank) with every rank on the one
    GPU over gloo: barrier + MAX-over-ranks timing, per-rank e2e, rank 0 alone prints
    (timings meaningless: the ranks share a GPU; the probes are in the slow N = 2 test)."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus",
                        str(world), "--dist-backend", "gloo", "--device-mod", "1", *SMALL, "--e2e-steps", "1",
                        "--e2e-warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1  # rank 0 alone prints
    b = lines[0]
    assert b["n_gpus"] == world and b["metric"] == _metric() and b["scaling"] == "strong" and b["value"] > 0
    assert b["config"]["numrn"] == 1 << 22 and b["config"]["per_gpu"] == (1 << 22) // world
    assert b["config"]["parallelism"] == f"gid-shard{world}"
    assert b["gpu_launches"] == b["steps"]  # rank 0's own launches (one fused launch per step)
    e = b["e2e"]
    assert e["d2h_bytes_per_step"] == 8 * (1 << 22) * 200 and e["value"] > 0


@pytest.mark.slow
def test_bench_two_ranks_default_is_config4_and_5():
    """The driver's N = 2 launch with the DEFAULT workload (2 ranks sharing the one GPU over
    gloo): device-only BASELINE config 4 (2^28 total, 2^27 per rank x 1000), e2e config 5
    (2^28 x 100), and the e2e roofline against the all-ranks-concurrent D2H probe."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
                        "--dist-backend", "gloo", "--device-mod", "1", "--steps", "2", "--warmup", "3",
                        "--sustained-steps", "2", "--e2e-steps", "1", "--e2e-warmup", "0", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    b = lines[0]
    assert b["n_gpus"] == 2 and b["scaling"] == "strong"
    assert b["config"]["numrn"] == 1 << 28 and b["config"]["per_gpu"] == 1 << 27 and b["config"]["numiter"] == 1000
    assert b["config"]["workload"].startswith("BASELINE config 4")
    e = b["e2e"]
    assert e["workload"].startswith("BASELINE config 5") and e["numiter"] == 100
    assert e["d2h_bytes_per_step"] == 8 * (1 << 28) * 100
    pr = b["probes"]
    assert len(pr["d2h_pinned_concurrent_gbs_per_rank"]) == 2
    assert e["roofline"]["peak"] == pytest.approx(pr["d2h_pinned_concurrent_gbs_aggregate"])
    assert "all 2 rank(s) at once" in e["roofline"]["peak_source"]
