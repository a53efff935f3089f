#!/usr/bin/env python3
"""Device-only throughput sweep over kernel variants / grid caps / ring sizes (GPU box).

    python tools/sweep.py [--numrn 16777216] [--numiter 1000] [--reps 5] > out.jsonl

Each line: variant, grid_warps cap, ring slots, best/median GB/s of prng_init +
prng_generate(numiter) timed with CUDA events on the generation stream."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402


def run(h, numrn, numiter, reps, gen):
    for _ in range(2):
        P.prng_init(h)
        P.prng_generate(h, numiter)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(gen)
        P.prng_init(h)
        P.prng_generate(h, numiter)
        b.record(gen)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    gbs = [8 * numrn * numiter / (t * 1e-3) / 1e9 for t in ts]
    return max(gbs), statistics.median(gbs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--numrn", type=int, default=1 << 24)
    ap.add_argument("--numiter", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="all")
    ap.add_argument("--warps", default="0")
    ap.add_argument("--slots", default="0")
    ap.add_argument("--pads", default="0")
    ap.add_argument("--cta-warps", default="0")
    ap.add_argument("--chunks", default="0", help="PRNG_OPT_CHUNK_ITERS values")
    ap.add_argument("--orders", default="0", help="PRNG_OPT_PIECE_ORDER values")
    ap.add_argument("--epochs", default="0", help="PRNG_OPT_EPOCH_ITERS values (0 auto, -1 off)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
    vs = range(P.prng_kernel_variants()) if a.variants == "all" else [int(v) for v in a.variants.split(",")]
    for slots, pad, cw, ch, od, ep in [(int(s), int(p), int(c), int(l), int(o), int(e)) for s in a.slots.split(",")
                                       for p in a.pads.split(",") for c in a.cta_warps.split(",")
                                       for l in a.chunks.split(",") for o in a.orders.split(",")
                                       for e in a.epochs.split(",")]:
        for w in [int(x) for x in a.warps.split(",")]:
            for v in vs:
                h = P.prng_create(a.numrn, 0)
                P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
                P.prng_set_option(h, P.PRNG_OPT_KERNEL, v)
                P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, w)
                P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, slots)
                P.prng_set_option(h, P.PRNG_OPT_RING_PAD, pad)
                P.prng_set_option(h, P.PRNG_OPT_CTA_WARPS, cw)
                P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, ch)
                P.prng_set_option(h, P.PRNG_OPT_PIECE_ORDER, od)
                P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, ep)
                best, med = run(h, a.numrn, a.numiter, a.reps, gen)
                _, _, rs, _, _ = P.prng_device_ring(h)
                ran, ran_e = P.prng_last_launch(h)
                P.prng_destroy(h)
                print(json.dumps({"variant": P.prng_kernel_variant_name(v), "grid_warps": w, "slots": rs, "pad": pad, "cta_warps": cw,
                                  "numrn": a.numrn, "numiter": a.numiter, "chunk": ch, "order": od, "epoch": ep,
                                  "ran": P.prng_kernel_variant_name(ran), "ran_epoch": ran_e,
                                  "best_gbs": round(best, 1), "median_gbs": round(med, 1)}), flush=True)


if __name__ == "__main__":
    main()
