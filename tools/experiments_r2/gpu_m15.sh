#!/bin/bash
# round 2, call m15: time-parallel launches at 8 warps/SM, one unit per warp -- Fig. 4 grid + GPU tests
O=gpurun_out/m15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/fig4_grid.py > $O/fig4.jsonl 2> $O/fig4.err
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" -k "time_parallel or chunk or randomised or epoch or anti_absorption or autotune or star" > $O/pytest_tp.log 2>&1; echo "rc=$?" >> $O/pytest_tp.log
