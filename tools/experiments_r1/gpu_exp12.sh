#!/bin/bash
OUT=gpurun_out/exp12; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
timeout 900 python tools/sweep.py --variants all --warps 0,296,592,888,1184,2368 --reps 3 > $OUT/s24.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,1,2,3,4,5,6 --warps 0,592,1184 --numrn 1048576 --reps 3 > $OUT/s20.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,1,2,3,4,5,6 --warps 0,592,1184 --numrn 268435456 --numiter 100 --reps 3 > $OUT/s28.jsonl 2>&1
python -c "
import paper_1609_01257_b200 as P, torch
torch.cuda.set_device(0)
print('memset 32GiB', P.prng_probe_memset_gbs(32<<30, 3))
print('store 32GiB', P.prng_probe_store_gbs(32<<30, 3))
print('memset 4GiB', P.prng_probe_memset_gbs(4<<30, 3))
print('store 4GiB', P.prng_probe_store_gbs(4<<30, 3))
" > $OUT/probes.txt 2>&1
