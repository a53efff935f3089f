#!/bin/bash
# round 2, call m9: sustained (power-capped) A/B of grid shapes and variants at the bench shape
O=gpurun_out/m9; mkdir -p $O
timeout 900 python tools/sustained.py "v4n8s1a:0:0,v4n8s1a:1184:8,v4n8s1a:1184:4,v4n4s1p:0:0,v4n16s1:0:0,v2n4s1:0:0,v4n8s1:0:0,v4n8s1a:296:2" 3 50 > $O/sustained.jsonl 2> $O/sustained.err
