#!/bin/bash
# run-to-run variance of the bench line, and the e2e pipeline modes at the full config-3 shape
OUT=gpurun_out/var; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for r in 1 2 3; do timeout 600 python bench.py --no-cpu > $OUT/bench_$r.json 2> $OUT/bench_$r.err; done
for m in 0 1 2 3 4; do timeout 900 python bench.py --no-cpu --no-probes --steps 1 --warmup 1 --e2e-steps 1 --e2e-mode $m > $OUT/e2e_mode$m.json 2> $OUT/e2e_mode$m.err; done
