#!/bin/bash
OUT=gpurun_out/exp10; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/sweep.py --variants 0,1,4 --slots 16,1000 --reps 3 > $OUT/bigring.jsonl 2>&1
timeout 600 ncu --metrics dram__bytes_write.sum,dram__cycles_active_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:batch -s 2 -c 1 --log-file $OUT/dram_bigring.csv python tools/sweep.py --variants 0 --slots 1000 --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_write.sum,dram__cycles_active_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:batch -s 2 -c 1 --log-file $OUT/dram_ring16.csv python tools/sweep.py --variants 0 --slots 16 --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_write.sum,dram__cycles_active_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:batch -s 2 -c 1 --log-file $OUT/dram_v4n8_ring16.csv python tools/sweep.py --variants 4 --slots 16 --reps 1 > /dev/null 2>&1
