#!/bin/bash
OUT=gpurun_out/exp16; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "every_variant or ragged" > $OUT/pytest_gpu.log 2>&1
timeout 900 python tools/sweep.py --variants 0,12,15,16,17,18,19,20 --reps 3 > $OUT/s24.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,15,16,17,19,20 --numrn 1048576 --reps 3 > $OUT/s20.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,15,16,17,19,20 --numrn 268435456 --numiter 100 --reps 3 > $OUT/s28.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 15,16,17 --warps 296,1184,2368 --reps 3 > $OUT/s24w.jsonl 2>&1
