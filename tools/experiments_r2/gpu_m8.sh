#!/bin/bash
O=gpurun_out/m8; mkdir -p $O
G=tools/experiments_r2/gen_sched
$G 16777216 1000 > $O/s24_t1000.jsonl 2>&1
