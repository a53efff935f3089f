#!/bin/bash
# exp28: compute-sanitizer over every kernel family incl. the epoch kernel and the
# anti-absorption substitution (tools/sanitize_cases.py).
OUT=gpurun_out/exp28; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/sanitize_cases.py > $OUT/plain.txt 2>&1
for T in synccheck memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1
  echo "rc=$?" >> $OUT/san_$T.txt
done
ls -la $OUT
