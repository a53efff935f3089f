#!/bin/bash
OUT=gpurun_out/exp7; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "ragged or spec_grid or config1" > $OUT/pytest_gpu.log 2>&1
V=8,12,15,16,17,18
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --reps 3 > $OUT/s24.jsonl 2>&1
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --numrn 1048576 --reps 3 > $OUT/s20.jsonl 2>&1
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --numrn 4194304 --reps 3 > $OUT/s22.jsonl 2>&1
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --numrn 268435456 --numiter 100 --slots 4 --reps 3 > $OUT/s28.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 15,16,17 --warps 592,1184 --lag 1 --reps 3 > $OUT/s24lag1.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 15,16,17 --warps 592,1184 --lag 4 --reps 3 > $OUT/s24lag4.jsonl 2>&1
