#!/bin/bash
# one-shot grids with resident CTAs per SM capped by dynamic shared memory (experimental build)
O=gpurun_out/${1:-m37}; mkdir -p $O
F=paper_1609_01257_b200/csrc/prng_engine.cu
cp $F /tmp/engine_orig.cu
python tools/experiments_r2/occ_patch.py $F
python -c "from paper_1609_01257_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
for r in 1 2; do
  timeout 300 python tools/experiments_r2/occ_probe.py persistent 0 >> $O/occ.jsonl 2>> $O/occ.err
  timeout 300 python tools/experiments_r2/occ_probe.py oneshot-native 2 >> $O/occ.jsonl 2>> $O/occ.err
  for c in 2 3 4 6; do
    S=$(( (233472 / c) - 1024 - 2048 ))
    PRNG_EXP_SMEM=$S timeout 300 python tools/experiments_r2/occ_probe.py oneshot-cap$c 2 >> $O/occ.jsonl 2>> $O/occ.err
  done
done
cp /tmp/engine_orig.cu $F
