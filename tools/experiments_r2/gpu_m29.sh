#!/bin/bash
O=gpurun_out/${1:-m29}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/experiments_r2/tp_warps.py > $O/tp_warps.jsonl 2> $O/tp_warps.err
