#!/bin/bash
# ncu launch list + --set full of the bench kernel, current tree.
OUT=gpurun_out/${1:-ncu_final}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-probes > $OUT/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:batch_kernel -c 1 \
    -o $OUT/prof_batch python tools/profile_step.py > $OUT/ncu_full.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
ls -la $OUT
