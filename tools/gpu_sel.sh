#!/bin/bash
O=gpurun_out/${1:-sel}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "$2" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
