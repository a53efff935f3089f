#!/bin/bash
# per-DRAM-channel activity (ncu metric instances) of the generator vs the one-shot fill
O=gpurun_out/${1:-m28}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --metrics dram__cycles_active.sum,dram__cycles_active.min,dram__cycles_active.max,dram__cycles_elapsed.max,dram__bytes_write.sum,dram__bytes_write.min,dram__bytes_write.max,dram__bytes_read.sum,gpu__time_duration.sum \
   --print-metric-instances values --clock-control none --csv -k regex:"batch_kernel|fill_probe" \
   python tools/experiments_r2/chan_probe.py > $O/chan.csv 2> $O/chan.err
