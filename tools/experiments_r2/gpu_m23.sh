#!/bin/bash
# fused a1: GPU suite (fast), smoke, small-n costs, bench
O=gpurun_out/${1:-m23}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $O/pytest_gpu_fast.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_fast.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python tools/experiments_r2/small_cost.py > $O/small_cost.jsonl 2> $O/small_cost.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
