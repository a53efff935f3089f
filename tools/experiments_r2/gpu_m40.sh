#!/bin/bash
O=gpurun_out/${1:-m40}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/experiments_r2/oneshot_sustained_ab.py > $O/sust_ab.jsonl 2> $O/sust_ab.err
