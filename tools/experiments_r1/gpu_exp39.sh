#!/bin/bash
# exp39: numrn = 2^28 x 1000 on one GPU (32 ring slots): epoch order (auto) vs v2n32s1 in
# natural order at 4 and 8 warps per SM (live set 155 / 310 MB), with ncu DRAM bytes.
OUT=gpurun_out/exp39; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
S="timeout 900 python tools/sweep.py --reps 3 --numrn $((1 << 28)) --numiter 1000"
$S --variants 0 >> $OUT/n28.jsonl 2>> $OUT/err.log
$S --variants 14 --warps 592,1184 >> $OUT/n28.jsonl 2>> $OUT/err.log
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum"
cat > /tmp/p39.py <<'PY'
import os, sys
sys.path.insert(0, ".")
import paper_1609_01257_b200 as P
h = P.prng_create(1 << 28, 0)
P.prng_set_option(h, P.PRNG_OPT_KERNEL, 14)
P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, int(os.environ["W"]))
P.prng_init(h); P.prng_generate(h, 1000); P.prng_destroy(h)
PY
for w in 592 1184; do
  W=$w timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv python /tmp/p39.py > $OUT/ncu_w$w.csv 2>> $OUT/err.log
done
ls -la $OUT
