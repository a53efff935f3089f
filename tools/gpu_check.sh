#!/bin/bash
# One gpurun call: build, GPU tests (fast, then slow), smoke, bench, reference arm, ncu launch
# list + full capture of the top kernel.
# Usage (from the repo root, on the GPU box): bash tools/gpu_check.sh [tag] [skip-slow]
set -x
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/pytest_gpu_fast.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_fast.log
if [ -z "$2" ]; then
  timeout 2400 python -m pytest tests -q -m "gpu and slow" --durations=0 > $OUT/pytest_gpu_slow.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_slow.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# ncu: the default variant (id 0) in bench.py's launch configuration
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --kernel 0 --steps 2 --warmup 1 --no-e2e --no-cpu --no-probes --sustained-steps 0 > $OUT/ncu_launches.log 2>&1
# full section set: application replay (no 64 GiB save/restore per pass)
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:batch_kernel -c 1 \
    -o $OUT/prof_batch python tools/profile_step.py > $OUT/ncu_full.log 2>&1
ls -la $OUT
