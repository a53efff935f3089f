#!/bin/bash
# exp33: interleaved CTA vectors (v4n8s1ai) vs v4n8s1a at the bench shape; parity of all variants.
OUT=gpurun_out/exp33; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_variant or randomised or ragged or time_parallel" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for round in 1 2 3; do
  for k in 30 34; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
ls -la $OUT
