#!/bin/bash
# BASELINE configs 4 and 5 at their per-rank shapes on one GPU (P = 8, 4, 2, 1 ranks of 2^28).
OUT=gpurun_out/${1:-cfg}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for lg in 25 26 27 28; do
  timeout 600 python bench.py --numrn-total $((1<<lg)) --numiter 1000 --steps 3 --warmup 3 --no-e2e --no-cpu --no-probes --sustained-steps 0 > $OUT/c4_2p$lg.json 2> $OUT/c4_2p$lg.err
done
timeout 600 python bench.py --numrn-total $((1<<25)) --numiter 1000 --e2e-numiter 100 --steps 3 --warmup 3 --e2e-steps 2 --no-cpu --no-probes --sustained-steps 0 > $OUT/c5_2p25.json 2> $OUT/c5_2p25.err
# ncu DRAM bytes of the per-rank config-4 launches (the anti-absorption rule's variants)
for lg in 25 26 27; do
  PRNG_N=$((1<<lg)) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:batch_kernel -c 1 --csv --log-file $OUT/ncu_c4_2p$lg.csv python tools/profile_step.py > /dev/null 2>&1
done
