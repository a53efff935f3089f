#!/bin/bash
O=gpurun_out/${1:-m31}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/experiments_r2/mid_warps.py > $O/mid_warps.jsonl 2> $O/mid_warps.err
