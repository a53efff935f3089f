#!/bin/bash
# exp17: why does numrn = 2^28 x 100 reach the memset fill rate (7.44 TB/s) while the bench
# shape 2^24 x 1000 stops at ~6.9?  (a) numrn / iterations per launch, (b) forced
# jump-started chunks (rounds of L iterations at 2^24), (c) CTA-blocked piece order.
OUT=gpurun_out/exp17
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forced" > $OUT/pytest_forced.log 2>&1
echo "rc=$?" >> $OUT/pytest_forced.log
S="timeout 600 python tools/sweep.py --variants 0 --reps 5"
for n in 24 25 26 27 28; do
  for i in 100 1000; do
    $S --numrn $((1 << n)) --numiter $i >> $OUT/sizes.jsonl 2>> $OUT/err.log
  done
done
$S --chunks 0,25,50,100,250,500 --orders 0,1 >> $OUT/chunks_2e24.jsonl 2>> $OUT/err.log
$S --numrn $((1 << 28)) --numiter 100 --orders 0,1 >> $OUT/order_2e28.jsonl 2>> $OUT/err.log
$S --chunks 0,100 --orders 0,1 --warps 592,1184 >> $OUT/chunks_warps_2e24.jsonl 2>> $OUT/err.log
# memset in the same run
python - >> $OUT/memset.txt 2>&1 <<'EOF'
import paper_1609_01257_b200 as P
import torch; torch.cuda.set_device(0)
print("memset_gbs", P.prng_probe_memset_gbs(32 << 30))
EOF
ls -la $OUT
