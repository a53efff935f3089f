#!/bin/bash
# exp38: die-locality probe (tools/experiments_r1/die_probe.cu).
OUT=gpurun_out/exp38; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/die_probe tools/experiments_r1/die_probe.cu > $OUT/build.log 2>&1
timeout 300 /tmp/die_probe lat $OUT/groups.bin > $OUT/lat.txt 2>&1
timeout 300 /tmp/die_probe lat $OUT/groups2.bin > $OUT/lat2.txt 2>&1
timeout 600 /tmp/die_probe write $OUT/groups.bin > $OUT/write.txt 2>&1
ls -la $OUT
