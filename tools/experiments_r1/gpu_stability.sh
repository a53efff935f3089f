#!/bin/bash
# Stability: the full GPU suite twice and bench.py three times on one box (flakiness and
# run-to-run spread of the headline numbers).
OUT=gpurun_out/${1:-stability}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2; do
  timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$i.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$i.log
done
for i in 1 2 3; do
  timeout 900 python bench.py > $OUT/bench_$i.json 2> $OUT/bench_$i.err
done
ls -la $OUT
