#!/bin/bash
OUT=gpurun_out/exp1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/sweep.py --warps 0,1184,2368,9472 > $OUT/sweep_warps.jsonl 2>&1
timeout 300 python tools/sweep.py --variants 0,4,5 --slots 2,4,16,64 > $OUT/sweep_slots.jsonl 2>&1
timeout 300 ncu --metrics dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_op_write.sum,launch__grid_size,launch__block_size --csv --log-file $OUT/calib.csv python tools/calib_dram.py 32 > $OUT/calib.log 2>&1
