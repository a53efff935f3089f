#!/bin/bash
# exp37: ping-pong form of the wide variants at the C4 per-rank shapes (honest live sets).
OUT=gpurun_out/exp37; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_variant" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for round in 1 2; do
  timeout 900 python tools/sweep.py --reps 3 --numrn $((1 << 26)) --numiter 1000 --variants 17,36 >> $OUT/n26.jsonl 2>> $OUT/err.log
  timeout 900 python tools/sweep.py --reps 3 --numrn $((1 << 27)) --numiter 1000 --variants 14,37 >> $OUT/n27.jsonl 2>> $OUT/err.log
  timeout 900 python tools/sweep.py --reps 3 --numrn $((1 << 25)) --numiter 1000 --variants 30,34 >> $OUT/n25.jsonl 2>> $OUT/err.log
done
ls -la $OUT
