#!/bin/bash
O=gpurun_out/${1:-m39}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python tools/experiments_r2/oneshot_variant.py > $O/variant.jsonl 2> $O/variant.err
