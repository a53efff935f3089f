#!/bin/bash
# Closing check of a session: build, the whole GPU suite (fast + slow), smoke, bench
# (+ reference arm) at the driver's 20 / 5 steps, ncu
# launch list + --set full capture of the bench kernel.
# Usage (repo root, on the GPU box): bash tools/gpu_close.sh TAG
set -x
OUT=gpurun_out/${1:-close}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -q -m "gpu and not slow" > $OUT/pytest_gpu_fast.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_fast.log
timeout 2400 python -m pytest tests -q -m "gpu and slow" --durations=0 > $OUT/pytest_gpu_slow.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_slow.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
# compute-sanitizer is closed on this GPU pool (r2q: it refuses to run, rc 86); the
# sanitizer cases stay in tools/sanitize_cases.py / tools/gpu_san.sh for pools that allow it.
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --kernel 0 --steps 2 --warmup 1 --no-e2e --no-cpu --no-probes --sustained-steps 0 > $OUT/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:batch_kernel -c 1 \
    -o $OUT/prof_batch python tools/profile_step.py > $OUT/ncu_full.log 2>&1
ls -la $OUT
