#!/bin/bash
O=gpurun_out/m17; mkdir -p $O
timeout 900 python tools/experiments_r2/small_variant_ab.py > $O/ab.jsonl 2> $O/ab.err
