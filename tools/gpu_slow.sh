#!/bin/bash
O=gpurun_out/${1:-slow}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
free -g > $O/free.txt 2>&1
timeout 2400 python -m pytest tests -q -m "gpu and slow" --durations=0 > $O/pytest_gpu_slow.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_slow.log
