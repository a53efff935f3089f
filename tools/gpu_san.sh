#!/bin/bash
# GPU tests (fast) + compute-sanitizer (4 tools) over tools/sanitize_cases.py
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -q -m "gpu and not slow" > $OUT/pytest_gpu_fast.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_fast.log
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1; echo "rc=$?" >> $OUT/san_$T.txt
done
