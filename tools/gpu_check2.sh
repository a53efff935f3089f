#!/bin/bash
OUT=gpurun_out/chk2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1
done
