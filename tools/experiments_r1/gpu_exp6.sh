#!/bin/bash
OUT=gpurun_out/exp6; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
V=8,12,13,14,15,16,17,18,19,20
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --reps 3 > $OUT/s24.jsonl 2>&1
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --numrn 1048576 --reps 3 > $OUT/s20.jsonl 2>&1
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --numrn 4194304 --reps 3 > $OUT/s22.jsonl 2>&1
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --numrn 268435456 --numiter 100 --slots 4 --reps 3 > $OUT/s28.jsonl 2>&1
