#!/bin/bash
O=gpurun_out/m16; mkdir -p $O
timeout 600 python tools/experiments_r2/tp_ab.py > $O/tp_ab.jsonl 2> $O/tp_ab.err
