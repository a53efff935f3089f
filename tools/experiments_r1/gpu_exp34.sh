#!/bin/bash
# exp34: compute-sanitizer over the extended case list (session-2 variants included).
OUT=gpurun_out/exp34; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/sanitize_cases.py > $OUT/plain.txt 2>&1
for T in synccheck racecheck memcheck; do
  timeout 1500 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1; echo "rc=$?" >> $OUT/san_$T.txt
done
ls -la $OUT
