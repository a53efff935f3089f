#!/bin/bash
OUT=gpurun_out/exp9; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "zerocopy or host_memory or pipeline_modes" > $OUT/pytest_gpu.log 2>&1
timeout 900 python tools/e2e_sweep.py > $OUT/e2e.jsonl 2>&1
for IT in 16 32 64 128; do
timeout 300 ncu --metrics dram__bytes_write.sum,dram__sectors_write.sum,fbpa__dram_write_bytes.sum,lts__t_sectors_op_write.sum,dram__cycles_active_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/dram_it$IT.csv python bench.py --kernel 0 --numiter $IT --steps 1 --warmup 0 --no-e2e --no-cpu --no-probes > /dev/null 2>&1
done
