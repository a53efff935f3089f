#!/bin/bash
OUT=gpurun_out/exp11; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/sweep.py --variants 0 --slots 16,32,64,128,256,512,1000 --reps 3 > $OUT/rings.jsonl 2>&1
for S in 32 64 128 256 512; do
timeout 600 ncu --metrics dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_l1_op_write_lookup_hit.sum,lts__t_sectors_srcunit_l1_op_write_lookup_miss.sum --clock-control none --csv \
    -k regex:batch -s 2 -c 1 --log-file $OUT/dram_s$S.csv python tools/sweep.py --variants 0 --slots $S --reps 1 > /dev/null 2>&1
done
