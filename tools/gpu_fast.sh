#!/bin/bash
O=gpurun_out/${1:-fast}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $O/pytest_gpu_fast.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_fast.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
