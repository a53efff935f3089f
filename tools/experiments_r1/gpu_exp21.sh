#!/bin/bash
# exp21: epoch kernel state-load kinds (29 = .cg prefetch, 0 = weak prefetch [default],
# 30 = weak load at unit start) vs natural order, 2^24 (forced E) and 2^27 (auto E = 64).
OUT=gpurun_out/exp21
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
S="timeout 900 python tools/sweep.py --reps 5 --numiter 1000"
$S --variants 0,29,30 --numrn $((1 << 24)) --epochs=-1,256,64 >> $OUT/e_2e24.jsonl 2>> $OUT/err.log
$S --variants 0,29,30 --numrn $((1 << 27)) --epochs=0 >> $OUT/e_2e27.jsonl 2>> $OUT/err.log
$S --variants 3,2,1 --numrn $((1 << 27)) --epochs=0 >> $OUT/e_2e27.jsonl 2>> $OUT/err.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "epoch" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
ls -la $OUT
