#!/bin/bash
O=gpurun_out/${1:-m22}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/experiments_r2/small_cost.py > $O/small_cost.jsonl 2> $O/small_cost.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python tools/experiments_r2/small_cost.py > /dev/null 2>&1
