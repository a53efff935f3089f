#!/bin/bash
# exp41: 2-CTA cluster barrier on the bench geometry (v4n8c2) vs v4n8s1a.
OUT=gpurun_out/exp41; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_variant" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for round in 1 2 3; do
  for k in 31 14; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
ls -la $OUT
