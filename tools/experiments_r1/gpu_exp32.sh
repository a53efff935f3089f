#!/bin/bash
# exp32: CTA-coherent TMA bulk stores (c4n8s3 / c4n8s4) vs the bench kernel (v4n8s1a).
OUT=gpurun_out/exp32; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_variant" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for round in 1 2 3; do
  for k in 30 38 39; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed"
PRNG_KERNEL=39 timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv python tools/profile_step.py > $OUT/ncu_k39.csv 2>> $OUT/err.log
ls -la $OUT
