#!/usr/bin/env python3
"""bench.py -- massive-PRNG hot path (arXiv 1609.01257 §5) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] ...
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One "step" = one pass of the whole hot path over one synthetic workload:
prng_init (a1, seeding kernel) + prng_generate(numiter) (a2+a3: xorshift64 batch kernel,
register-resident state, 32-byte stores into a device ring).  BASELINE.json's metric is
random numbers/s (and GB/s, 8 B per number, Eq. 1) device-only and end to end.

* value      device-only numbers/s over all ranks: inputs (numrn, numiter, seed) resident,
             output through a 64 GiB rotating ring in HBM (no address rewritten within
             64 GiB, > 500x the 126 MB L2, so no L2 flush is needed).
             Timed with CUDA events on the generation stream (a torch stream handed to the
             library), K steps between barrier + synchronize, max over ranks.
* e2e        same metric through the C-ABI call with HOST buffers: prng_generate with the
             null sink (the paper discards stdout), i.e. device ring -> D2H on a side
             stream -> pinned host double buffer -> sink, all inside the timed region.
* roofline   dominant kernel (the batch kernel): algorithmic bytes per launch
             (8 B x numbers) / mean launch duration from CUDA events on its stream,
             against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline  the oracle (oracle/, plain single-threaded C) on a bounded sample.

Rank r of N owns the contiguous gid range shard_range(numrn_total, r, N) (weak scaling:
numrn per GPU fixed, default 2^24).  The only collectives are a barrier and a MAX
all-reduce of the elapsed times.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json "metric", verbatim: `value` is its device-only numbers/s (8 B per number),
# `e2e` its end-to-end D2H figure, `roofline` the "vs roofline" part.
METRIC = "random numbers/s (GB/s) device-only and end-to-end D2H at 1/2/4/8 B200 vs roofline"
METRIC_DETAIL = "value: device-only random numbers/s (gbs = 8 B/number); e2e: same through host buffers"

from workloads import SEED_PERF, shard_range  # noqa: E402

HBM_THEORETICAL_GBS = 8 * 1024 / 8 * 2 * 3.996  # 8 HBM3e stacks x 1024 bit x 2 x 3996 MHz
DEF_NUMRN = 1 << 24
DEF_NUMITER = 1000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--numrn-per-gpu", type=int, default=DEF_NUMRN)
    ap.add_argument("--numrn-total", type=int, default=0, help="strong scaling: fixed total numrn (e.g. 2^28)")
    ap.add_argument("--numiter", type=int, default=DEF_NUMITER)
    ap.add_argument("--seed", type=int, default=SEED_PERF)
    ap.add_argument("--kernel", type=int, default=0, help="kernel variant id (default 0 = auto: v4n8s1 at the bench shape; -1: prng_autotune)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--e2e-mode", type=int, default=3, help="0 S0, 1 S1, 2 O1, 3 O2, 4 O3 (zero-copy)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-probes", action="store_true")
    ap.add_argument("--cpu-numiter", type=int, default=64, help="oracle sample: numiter at full numrn")
    ap.add_argument("--ref-numiter", type=int, default=8, help="--impl reference: numiter per step sample")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--output", type=int, default=0, help="0 = the state (paper); 1 = xorshift64* scrambled (NEXT-3)")
    ap.add_argument("--no-numa-bind", action="store_true", help="keep the process's CPU affinity")
    ap.add_argument("--device-mod", type=int, default=0,
                    help="TEST ONLY: map local rank r to GPU r %% K (several ranks per GPU; timings meaningless)")
    return ap.parse_args()


# ---------------------------------------------------------------- distributed plumbing
class Dist:
    def __init__(self, backend):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = None
        if self.world > 1 and backend:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist:
            if self.dist.get_backend() == "nccl":  # name the device: no guess by NCCL
                import torch
                self.dist.barrier(device_ids=[torch.cuda.current_device()])
            else:
                self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        dev = "cuda" if self.dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------- clocks during timing
class Clocks:
    """SM clock + clock-event reasons sampled every 5 ms by NVML (nvidia_ml_py) in a thread
    while the timed region runs (B200_PROFILING.md's clocks line; nvidia-smi would need
    ~0.5 s to start, longer than the ~100 ms device-only timed region).  Samples taken
    while the GPU is idle (GpuIdle reason) are excluded from the median."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.rows.append(self._sample())
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        return self

    def _sample(self):
        N = self.N
        return (N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM), N.nvmlDeviceGetCurrentClocksEventReasons(self.h))

    def _loop(self):
        while not self.stop.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:  # noqa: BLE001
                pass
            self.stop.wait(0.005)

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)
            self.rows.append(self._sample())

    def summary(self):
        if not self.t:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: " + getattr(self, "err", "")]}
        N = self.N
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap,
                "hw_power_brake_slowdown": N.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        busy = [(c, r) for c, r in self.rows if not (r & N.nvmlClocksEventReasonGpuIdle)] or self.rows
        reasons = sorted({nm for _, r in busy for nm, b in bits.items() if r & b})
        return {"sm_mhz": statistics.median(c for c, _ in busy), "sm_max_mhz": self.max, "reasons": reasons,
                "samples": len(self.rows), "busy_samples": len(busy), "source": "nvml 5 ms"}


def bind_to_gpu_cpus(dev):
    """Pin this rank to the CPUs NVML reports as local to its GPU, before any pinned host
    buffer is allocated, so the D2H targets NUMA-local memory."""
    try:
        import pynvml as N
        N.nvmlInit()
        hd = N.nvmlDeviceGetHandleByIndex(dev)
        ncpu = os.cpu_count() or 1
        words = N.nvmlDeviceGetCpuAffinity(hd, (ncpu + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(ncpu))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return {"cpus": len(cpus), "of": ncpu}
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)}
    return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy, read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(variant, epoch):
    """Per-launch DRAM bytes of the batch kernel from the committed ncu --set full summary,
    if that capture is of this kernel (variant "v{VEC}n{NPT}s1[a]", natural order)."""
    import re
    p = os.path.join(ROOT, "profiles", "ncu_batch_kernel.json")
    m = re.fullmatch(r"v(\d+)n(\d+)s1(a?)", variant or "")
    if not os.path.exists(p) or not m or epoch:
        return None, None
    with open(p) as f:
        d = json.load(f)
    # ncu spells bools as 0/1; later template parameters (IL, PP) default to 0
    want = [m.group(1), m.group(2), "0", "1", "0", "1" if m.group(3) else "0"]

    def same_kernel(name):
        mm = re.search(r"batch_kernel<([^>]*)>", name)
        if not mm:
            return False
        args = [x.strip() for x in mm.group(1).split(",")]
        return args[:6] == want and all(x in ("0", "false") for x in args[6:])

    if not any(same_kernel(k.get("kernel", "")) for k in d.get("kernels", [])):
        return None, None
    return d.get("dram_bytes_per_launch"), d.get("algorithmic_bytes_per_launch")


# ---------------------------------------------------------------- oracle timing (CPU)
def cpu_baseline(numrn, numiter, seed):
    import oracle
    t = time.perf_counter()
    oracle.digest(numrn, numiter, seed)
    dt = time.perf_counter() - t
    return numrn * numiter / dt, dt


def cpu_baseline_all_cores(numrn, numiter, seed):
    """The same oracle function, unchanged, on one contiguous gid shard per host core
    (threads: ctypes releases the GIL), as BASELINE.md's CPU plan asks."""
    import threading
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.lib()
    shards = [shard_range(numrn, r, cores) for r in range(cores)]
    th = [threading.Thread(target=oracle.digest, args=(numrn, numiter, seed, b, c)) for b, c in shards if c]
    t = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t
    return numrn * numiter / dt, dt, len(th)


def run_reference(a, D):
    """--impl reference: the oracle as it stands, on the host cores, rank 0 only."""
    if D.rank != 0:
        return
    import oracle
    oracle.build()
    numrn = a.numrn_total or a.numrn_per_gpu * D.world
    ni = a.ref_numiter
    for _ in range(a.warmup):
        oracle.digest(numrn, ni, a.seed)
    t = time.perf_counter()
    for _ in range(a.steps):
        oracle.digest(numrn, ni, a.seed)
    dt = time.perf_counter() - t
    v = numrn * ni * a.steps / dt
    sample = f"numrn={numrn} x numiter={ni} per step (of the workload's numiter={a.numiter}); digest-folded"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "metric_detail": METRIC_DETAIL, "value": v,
        "unit": "numbers/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"numrn={numrn}, numiter={a.numiter}, seed={a.seed} (sampled)"},
        "cpu_baseline": {"value": v, "unit": "numbers/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "numbers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(a, D):
    import torch
    import paper_1609_01257_b200 as P

    dev = D.local % a.device_mod if a.device_mod > 0 else D.local
    torch.cuda.set_device(dev)
    numa = bind_to_gpu_cpus(dev) if not a.no_numa_bind else None
    numrn = a.numrn_total or a.numrn_per_gpu * D.world
    gb, cnt = shard_range(numrn, D.rank, D.world)
    gen = torch.cuda.Stream()
    cop = torch.cuda.Stream()
    h = P.prng_create_range(numrn, a.seed, gb, cnt, dev)
    P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
    P.prng_set_option(h, P.PRNG_OPT_MODE, a.e2e_mode)
    P.prng_set_option(h, P.PRNG_OPT_OUTPUT, a.output)
    tune_gbs = None
    if a.kernel < 0:  # untimed setup, like a library autotuner; off by default so
        # the timed kernel is the one profiles/ holds the ncu capture of
        tune_gbs = P.prng_autotune(h)
    else:
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, a.kernel)
    kernel = P.prng_get_option(h, P.PRNG_OPT_KERNEL)
    grid_warps = P.prng_get_option(h, P.PRNG_OPT_GRID_WARPS)

    # ---- device only
    for _ in range(a.warmup):
        P.prng_init(h)
        P.prng_generate(h, a.numiter)
    # Timed region: K steps enqueued back to back on the generation stream (no host round
    # trips between steps: PRNG_OPT_BLOCKING 0), per-launch CUDA-event intervals accumulated
    # (PRNG_OPT_PROFILE 2) and read after the region.
    def timed_region():
        P.prng_set_option(h, P.PRNG_OPT_PROFILE, 2)
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(dev) as clk:
            D.barrier()
            torch.cuda.synchronize()
            ev0.record(gen)
            for _ in range(a.steps):
                P.prng_init(h)
                P.prng_generate(h, a.numiter)
            ev1.record(gen)
            torch.cuda.synchronize()
            D.barrier()
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 1)
        ids, s, e, _ = P.prng_prof_events(h)  # per-launch CUDA-event intervals of the K steps
        P.prng_set_option(h, P.PRNG_OPT_PROFILE, 0)
        return ev0.elapsed_time(ev1), ids, s, e, clk.summary()

    ms, ids, s, e, clocks = timed_region()
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake_slowdown"}
    # the contract: a run that saw these is rejected and re-measured once (decided jointly:
    # every rank takes part in the barriers of the re-run)
    if D.max(1.0 if bad & set(clocks["reasons"]) else 0.0) > 0:
        first = clocks
        ms, ids, s, e, clocks = timed_region()
        clocks["remeasured_after"] = first["reasons"]
    kern_ms = [1e3 * (y - x) for i, x, y in zip(ids, s, e) if i == 1]
    init_ms = [1e3 * (y - x) for i, x, y in zip(ids, s, e) if i == 0]
    launches = len(ids)
    ms_max = D.max(ms)
    numbers = numrn * a.numiter * a.steps
    value = numbers / (ms_max * 1e-3)

    peak, peak_src = measured_peaks()
    kmean = statistics.mean(kern_ms)
    algo_bytes = 8 * cnt * a.numiter
    achieved = algo_bytes / (kmean * 1e-3) / 1e9
    ran, epoch = P.prng_last_launch(h)  # the kernel the timed launches ran ("auto", anti-absorption)
    traffic, traffic_algo = ncu_traffic(P.prng_kernel_variant_name(ran), epoch)
    if traffic_algo is not None and int(traffic_algo) != algo_bytes:
        traffic = None  # the committed capture is of another shape
    kname = ("prngk::batch_kernel_epoch<" + P.prng_kernel_variant_name(ran) + f", E={epoch}>" if epoch else
             "prngk::batch_kernel<" + P.prng_kernel_variant_name(ran) + ">")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname,
                "grid_warps": grid_warps or "variant default", "autotune_probe_gbs": tune_gbs,
                "algorithmic_bytes_per_launch": algo_bytes, "mean_launch_ms": kmean,
                "kernel_share_of_step": sum(kern_ms) / ms, "init_kernel_mean_ms": statistics.mean(init_ms),
                "peak_source": peak_src,
                "frac_of_theoretical_hbm3e": achieved / HBM_THEORETICAL_GBS,
                "note": "write-only stream: the copy-based peak pays read/write turnarounds a pure write "
                        "stream does not; theoretical = 8 stacks x 1024 bit x 7.992 Gb/s = 8184 GB/s"}

    # ---- end to end (host buffers, D2H inside the timed region)
    e2e = None
    if not a.no_e2e:
        for _ in range(a.e2e_warmup):
            P.prng_init(h)
            P.prng_generate(h, a.numiter, P.SINK_NULL)
        walls = []
        for _ in range(a.e2e_steps):
            D.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.prng_init(h)
            P.prng_generate(h, a.numiter, P.SINK_NULL)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        # one more, untimed, step with per-batch CUDA-event intervals for the a6 overlap report
        P.prng_set_option(h, P.PRNG_OPT_PROFILE, 1)
        P.prng_init(h)
        P.prng_generate(h, a.numiter, P.SINK_NULL)
        prof = P.prng_prof_events(h)
        P.prng_set_option(h, P.PRNG_OPT_PROFILE, 0)
        wall = D.max(sum(walls))
        ev = numrn * a.numiter * a.e2e_steps / wall
        ids, s, e, w = prof
        calc = P.prng_prof_calc(ids, s, e, 4)
        agg = calc["agg"]
        ov = calc["overlap"]
        d2h_gbs = 8 * cnt * a.numiter * a.e2e_steps / sum(walls) / 1e9
        e2e = {"value": ev, "unit": "numbers/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": 8 * numrn * a.numiter, "gbs": 8 * ev / 1e9,
               "mode": ["S0", "S1", "O1", "O2", "O3"][a.e2e_mode], "d2h_gbs_per_gpu": d2h_gbs,
               "profile_extra_step": {
                   "rng_kernel_s": agg[1], "read_buffer_s": agg[2], "out_s": agg[3], "init_s": agg[0],
                   "rng_read_overlap_s": ov[1, 2],
                   "rng_hidden_frac": (ov[1, 2] / agg[1]) if agg[1] else None,
                   "copy_busy_frac": agg[2] / w if w else None, "effective_s": calc["effective"], "wall_s": w}}
        # the multi-rank form: D2H straight into a host array (ring of 2T rows, pinned by
        # torch), no staging buffer and no sink -- each rank writes its slice directly
        import numpy as np
        T = max(1, (256 << 20) // (8 * cnt))
        rows = 2 * T
        harr = torch.empty((rows, cnt), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        P.prng_init(h)
        P.prng_generate_host(h, min(a.numiter, rows), harr, cnt, rows)  # warm-up
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.prng_init(h)
        P.prng_generate_host(h, a.numiter, harr, cnt, rows)
        dt = D.max(time.perf_counter() - t0)
        e2e["host_array"] = {"value": numrn * a.numiter / dt, "unit": "numbers/s",
                             "gbs": 8 * numrn * a.numiter / dt / 1e9, "rows": rows,
                             "how": "prng_generate_host: D2H straight into a pinned host array (ring of rows)"}
        del harr
    probes = None
    if not a.no_probes and D.rank == 0:
        probes = {"memset_write_gbs": P.prng_probe_memset_gbs(32 << 30, 3),
                  "store_kernel_write_gbs": P.prng_probe_store_gbs(32 << 30, 3),
                  "d2h_pinned_gbs": P.prng_probe_d2h_gbs(1 << 30, 5, True, 1),
                  "d2h_pinned_2streams_gbs": P.prng_probe_d2h_gbs(1 << 30, 5, True, 2)}
        roofline["frac_of_same_box_memset"] = achieved / probes["memset_write_gbs"]
        roofline["frac_of_same_box_store_kernel"] = achieved / probes["store_kernel_write_gbs"]
        if e2e:
            e2e["roofline"] = {"bound": "host-link", "achieved": e2e["d2h_gbs_per_gpu"],
                               "peak": probes["d2h_pinned_gbs"], "unit": "GB/s",
                               "frac": e2e["d2h_gbs_per_gpu"] / probes["d2h_pinned_gbs"],
                               "peak_source": "same-box pinned cudaMemcpyAsync D2H 1 GiB, best of 5"}
    P.prng_destroy(h)

    cpu = None
    if D.rank == 0 and D.world == 1 and not a.no_cpu:
        v, dt = cpu_baseline(numrn, a.cpu_numiter, a.seed)
        cpu = {"value": v, "unit": "numbers/s", "cores": 1, "kind": "oracle",
               "sample": f"numrn={numrn} x numiter={a.cpu_numiter} ({dt:.1f} s, digest-folded, 1 thread)"}
        va, dta, nth = cpu_baseline_all_cores(numrn, 4 * a.cpu_numiter, a.seed)
        cpu["all_cores"] = {"value": va, "unit": "numbers/s", "cores": nth,
                            "sample": f"numrn={numrn} x numiter={4 * a.cpu_numiter} ({dta:.1f} s), one gid shard "
                                      f"per thread"}

    if D.rank == 0:
        line = {
            "metric": METRIC, "metric_detail": METRIC_DETAIL, "value": value, "unit": "numbers/s",
            "gbs": 8 * value / 1e9, "n_gpus": D.world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "strong" if a.numrn_total else "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (numrn, numiter, seed); outputs are the generated u64 stream",
            "config": {"workload": (f"BASELINE config 2: numrn=2^{numrn.bit_length() - 1} ({numrn}) per iteration"
                                    f" x numiter={a.numiter}, device-only" if D.world == 1 else
                                    f"numrn={numrn} total ({cnt} per GPU, gid-range sharded) x numiter={a.numiter}"),
                       "numrn": numrn, "numiter": a.numiter, "seed": a.seed, "parallelism": f"gid-shard{D.world}",
                       "output": ["state (paper)", "xorshift64* scrambled"][a.output],
                       "numa_bind": numa,
                       "l2": "output through a 64 GiB rotating ring per GPU (> 500x L2; no address rewritten "
                             "within 64 GiB, see profiles/r1_ring_absorption.md); no flush needed"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "probes": probes,
        }
        print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl != "reference" and a.dist_backend == "nccl":
        # bind this rank's GPU before the process group exists (NCCL uses the current device)
        import torch
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local % a.device_mod if a.device_mod > 0 else local)
    D = Dist(None if a.impl == "reference" else a.dist_backend)
    try:
        if a.impl == "reference":
            run_reference(a, D)
        else:
            run_ours(a, D)
    finally:
        D.close()


if __name__ == "__main__":
    main()
