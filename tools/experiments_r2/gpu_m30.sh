#!/bin/bash
O=gpurun_out/${1:-m30}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/experiments_r2/bimodal.py > $O/bimodal.jsonl 2> $O/bimodal.err
