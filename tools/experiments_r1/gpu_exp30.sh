#!/bin/bash
# exp30: barrier form made valid (.aligned only in uniform rounds, AL variants) --
# synccheck/racecheck, full GPU suite, smoke, bench-shape A/B, bench + reference, configs,
# launch list + ncu --set full of the bench kernel.
OUT=gpurun_out/exp30; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for T in synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1; echo "rc=$?" >> $OUT/san_$T.txt
done
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for round in 1 2 3; do
  for k in 3 30 29 31; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for lg in 25 26 27; do
  timeout 900 python bench.py --numrn-per-gpu $((1<<lg)) --numiter 1000 --steps 3 --warmup 3 --no-e2e --no-cpu --no-probes > $OUT/c4_2p$lg.json 2> $OUT/c4_2p$lg.err
done
timeout 900 python bench.py --numrn-per-gpu $((1<<25)) --numiter 100 --steps 3 --warmup 3 --e2e-steps 2 --no-cpu --no-probes > $OUT/c5_2p25.json 2> $OUT/c5_2p25.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-probes > $OUT/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:batch_kernel -c 1 \
    -o $OUT/prof_batch python tools/profile_step.py > $OUT/ncu_full.log 2>&1
ls -la $OUT
