#!/bin/bash
O=gpurun_out/${1:-m34}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/experiments_r2/oneshot_threshold.py > $O/threshold.jsonl 2> $O/threshold.err
timeout 1500 python -m pytest tests -q -m "gpu and not slow" -k "one_shot or auto_kernel or anti_absorption or fused or randomised" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
