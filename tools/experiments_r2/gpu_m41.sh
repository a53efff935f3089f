#!/bin/bash
O=gpurun_out/${1:-m41}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python tools/experiments_r2/pad_oneshot.py > $O/pad.jsonl 2> $O/pad.err

