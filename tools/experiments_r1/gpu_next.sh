#!/bin/bash
# NEXT rows on the GPU: tests, Fig. 3 summaries per pipeline mode, Fig. 5 chart, 2-rank bench flow.
OUT=gpurun_out/next1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
CLI=paper_1609_01257_b200/bin/rng_b200
for M in S0 S1 O1 O2 O3; do
  ( time timeout 300 $CLI 16777216 100 --mode $M --profile > /dev/null 2> $OUT/fig3_$M.txt ) 2> $OUT/time_$M.txt
  ( time timeout 300 $CLI 16777216 100 --mode $M --profile 2> $OUT/fig3_${M}_pipe.txt | cat > /dev/null ) 2> $OUT/time_${M}_pipe.txt
done
timeout 300 $CLI 16777216 8 --profile --export $OUT/fig5.tsv > /dev/null 2> $OUT/fig5_summary.txt
python tools/plot_events.py $OUT/fig5.tsv $OUT/fig5.svg --title "rng_b200 n=2^24 i=8 (O2): queue utilisation" 
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --dist-backend gloo --device-mod 1 --steps 2 --warmup 1 --no-cpu --no-probes --e2e-steps 1 --e2e-warmup 0 \
  > $OUT/bench_2rank_sharedgpu.json 2> $OUT/bench_2rank.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $OUT/bench_ref_2rank.json 2> $OUT/bench_ref_2rank.err
