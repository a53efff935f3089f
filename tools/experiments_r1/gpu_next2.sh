#!/bin/bash
OUT=gpurun_out/next2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py --output 1 --no-cpu --e2e-steps 1 > $OUT/bench_star.json 2> $OUT/bench_star.err
timeout 900 python tools/fig4_grid.py > $OUT/fig4.jsonl 2> $OUT/fig4.err
timeout 600 compute-sanitizer --tool memcheck --leak-check full python -c "import __graft_entry__ as g; g.smoke()" > $OUT/memcheck.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $OUT/racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $OUT/synccheck.txt 2>&1
