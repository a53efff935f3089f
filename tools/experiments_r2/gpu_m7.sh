#!/bin/bash
O=gpurun_out/m7; mkdir -p $O
timeout 600 tools/experiments_r2/colblock 16777216 256 > $O/colblock.jsonl 2>&1
