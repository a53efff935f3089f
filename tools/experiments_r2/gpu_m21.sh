#!/bin/bash
# sustained (power-capped) A/B: fewer SMs, fewer instructions per number
O=gpurun_out/${1:-m21}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=power.draw,clocks.sm --format=csv -lms 200 > $O/smi.csv 2>&1 &
SMI=$!
timeout 600 python tools/sustained.py "v4n8s1a:0:0,v4n8s1a:592:8,v4n8s1a:888:8,v4n8s1a:444:4,v4n4s1p:0:0,v4n8s1a:296:2" 3 100 > $O/sustained.jsonl 2> $O/sustained.err
kill $SMI
