#!/bin/bash
# fused a1 + 48-iteration chunks: GPU suite, smoke, small-n costs, Fig. 4 grid, bench
O=gpurun_out/${1:-m26}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -q -m "gpu and not slow" > $O/pytest_gpu_fast.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_fast.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python tools/experiments_r2/small_cost.py > $O/small_cost.jsonl 2> $O/small_cost.err
timeout 600 python tools/experiments_r2/tp_chunk_cells.py L48 > $O/cells.jsonl 2> $O/cells.err
timeout 900 python tools/fig4_grid.py > $O/fig4.jsonl 2> $O/fig4.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
