#!/bin/bash
# exp40: lean single-path kernel (v4n8s1l / v4n4s1l) vs v4n8s1a / v4n4s1p at the bench shape.
OUT=gpurun_out/exp40; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lean or every_variant or star_output_all or epoch_order" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for round in 1 2 3; do
  for k in 30 36 35 37; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
timeout 600 python tools/sustained.py v4n8s1a,v4n8s1l 6 50 > $OUT/sustained.jsonl 2>> $OUT/err.log
ls -la $OUT
