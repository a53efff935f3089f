#!/bin/bash
O=gpurun_out/${1:-m24}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/experiments_r2/short_chunks.py > $O/short_chunks.jsonl 2> $O/short_chunks.err
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $O/pytest_gpu_fast.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_fast.log
