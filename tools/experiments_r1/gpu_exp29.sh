#!/bin/bash
# exp29: CTA barrier form. Non-.aligned barrier.sync (valid PTX when the warps of a CTA
# reach it from different instructions) vs the round-1 .aligned bar.sync: synccheck over
# the sanitizer cases, then a bench-shape A/B (v4n8s1 / v4n8s1al, v4n4s1 / v4n4s1al).
OUT=gpurun_out/exp29; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > $OUT/san_synccheck.txt 2>&1; echo "rc=$?" >> $OUT/san_synccheck.txt
for round in 1 2 3; do
  for k in 3 30 29 31; do
    timeout 600 python bench.py --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu --no-probes >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
ls -la $OUT
