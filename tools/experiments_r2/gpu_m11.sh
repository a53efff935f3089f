#!/bin/bash
# round 2, call m11: sustained (~4 s each) memset vs one-shot fill vs the bench kernel, with NVML clocks
O=gpurun_out/m11; mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv &
SMI=$!
tools/experiments_r2/sustained_fill 32 800 > $O/fill.jsonl 2>&1
timeout 600 python tools/sustained.py "v4n8s1a:0:0" 2 200 > $O/kernel.jsonl 2> $O/kernel.err
kill $SMI
