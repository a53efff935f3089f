#!/bin/bash
# exp25: "auto" default (v4n8s1 from 2^21): full GPU suite, smoke, bench (+ reference),
# launch list and ncu --set full of the new bench kernel.
OUT=gpurun_out/exp25
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-probes > $OUT/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:batch_kernel -c 1 \
    -o $OUT/prof_batch python tools/profile_step.py > $OUT/ncu_full.log 2>&1
ls -la $OUT
