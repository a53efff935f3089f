#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over every kernel family
# (tools/sanitize_cases.py), then bench.py three times on the same box (stability).
OUT=gpurun_out/${1:-chk2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1; echo "rc=$?" >> $OUT/san_$T.txt
done
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err
done
ls -la $OUT
