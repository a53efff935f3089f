#!/bin/bash
# A/B of kTpMinChunk (128 = committed, then 64, 48, 32), two rounds each, on one box
O=gpurun_out/${1:-m25}; mkdir -p $O
F=paper_1609_01257_b200/csrc/prng_engine.cu
cp $F /tmp/engine_orig.cu
for rnd in 1 2; do
for L in 128 64 48 32; do
  sed "s/constexpr uint64_t kTpMinChunk = 128;/constexpr uint64_t kTpMinChunk = $L;/" /tmp/engine_orig.cu > $F
  python -c "from paper_1609_01257_b200 import _build; _build.build(force=True)" > $O/build_$L.log 2>&1
  timeout 600 python tools/experiments_r2/tp_chunk_cells.py "L$L" >> $O/cells.jsonl 2>> $O/cells.err
done
done
cp /tmp/engine_orig.cu $F
