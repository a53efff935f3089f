#!/bin/bash
# drift-bounded generator schedules (drift.cu)
O=gpurun_out/${1:-m18}; mkdir -p $O
D=tools/experiments_r2/drift
timeout 300 $D 16777216 1000 drift > $O/drift_spread.jsonl 2>&1
timeout 900 $D 16777216 1000 sweep > $O/sweep.jsonl 2>&1
