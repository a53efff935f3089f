#!/bin/bash
# A/B: e2e pipeline events created per call (build/ab/libprng_b200_head.so) vs the per-handle pool
O=gpurun_out/${1:-m27}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2; do
  timeout 600 python tools/experiments_r2/e2e_small.py head build/ab/libprng_b200_head.so >> $O/e2e_small.jsonl 2>> $O/e2e_small.err
  timeout 600 python tools/experiments_r2/e2e_small.py pool >> $O/e2e_small.jsonl 2>> $O/e2e_small.err
done
timeout 900 python -m pytest tests -q -m "gpu and not slow" -k "e2e or host or zerocopy or pipeline or sink or fused or profile" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
