#!/bin/bash
# Session-2 closing check on the committed tree: full GPU suite, smoke, bench (default),
# reference arm, a sustained bench (200 steps, power-capped), launch list.
OUT=gpurun_out/${1:-final_s2}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu --no-probes > $OUT/bench_sustained.json 2> $OUT/bench_sustained.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-probes > $OUT/ncu_launches.log 2>&1
ls -la $OUT
