#!/bin/bash
O=gpurun_out/m13; mkdir -p $O
timeout 600 python tools/experiments_r2/small_n.py > $O/small_n.jsonl 2> $O/small_n.err
