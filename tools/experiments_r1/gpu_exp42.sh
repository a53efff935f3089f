#!/bin/bash
# exp42: store cache policies on the bench kernel (v4n8s1a): default vs .cs / evict_first / no_allocate.
OUT=gpurun_out/exp42; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_variant" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for round in 1 2 3; do
  for k in 34 15 16 17; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
ls -la $OUT
