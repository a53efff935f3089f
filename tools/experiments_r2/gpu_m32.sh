#!/bin/bash
# One-shot (multi-wave) grids for the product kernel: an experimental build lifts the
# one-wave cap of max_grid_warps when PRNG_OPT_GRID_WARPS is set, so GRID_WARPS = all
# pieces gives one unit per warp (rounds = 1) and the hardware dispatches the CTAs in order.
O=gpurun_out/${1:-m32}; mkdir -p $O
F=paper_1609_01257_b200/csrc/prng_engine.cu
cp $F /tmp/engine_orig.cu
sed 's/        w = std::min<uint64_t>(w, (uint64_t)h->grid_warps);/        w = (uint64_t)h->grid_warps;  \/\/ EXPERIMENT: no one-wave cap/' /tmp/engine_orig.cu > $F
grep -n "EXPERIMENT" $F > $O/patch.txt
python -c "from paper_1609_01257_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
C="v4n8s1a:0:0,v4n8s1a:65536:4,v4n8s1a:65536:1,v4n8s1a:65536:2,v4n8s1a:65536:8,v4n4s1p:131072:4,v2n4s1:131072:4"
timeout 900 python tools/sustained.py "$C" 3 5 > $O/burst.jsonl 2> $O/burst.err
timeout 900 python tools/sustained.py "$C" 2 100 > $O/sustained.jsonl 2> $O/sustained.err
cp /tmp/engine_orig.cu $F
