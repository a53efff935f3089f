#!/bin/bash
O=gpurun_out/${1:-m36}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/experiments_r2/e2e_oneshot_ab.py > $O/e2e_ab.jsonl 2> $O/e2e_ab.err
