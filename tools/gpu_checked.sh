#!/bin/bash
# The kernels' own bounds checks (compute-sanitizer is closed on the GPU pool): build
# libprng_b200_checked.so (-DPRNG_CHECKED: every ring store / state access of the seed and
# batch kernels checked against its launch's arguments, trap on violation), then run the
# sanitizer cases and the fast GPU suite on it.  A trap fails the launch with a CUDA error
# and prints "prng bounds violation" with the address.
# Usage (repo root, on the GPU box): bash tools/gpu_checked.sh TAG
set -x
OUT=gpurun_out/${1:-checked}; mkdir -p $OUT
export PRNG_B200_CHECKED=1
python -c "from paper_1609_01257_b200 import _build; print(_build.build(force=True))" > $OUT/build.log 2>&1
timeout 600 python tools/sanitize_cases.py > $OUT/cases.txt 2>&1; echo "cases rc=$?" >> $OUT/cases.txt
timeout 2400 python -m pytest tests -q -m "gpu and not slow" -p no:cacheprovider > $OUT/pytest_gpu_fast.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_fast.log
timeout 2400 python -m pytest tests -q -m "gpu and slow" -p no:cacheprovider > $OUT/pytest_gpu_slow.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_slow.log
grep -l "bounds violation" $OUT/*.txt $OUT/*.log > $OUT/violations.txt 2>&1
echo "files with violations: $(wc -l < $OUT/violations.txt)" >> $OUT/violations.txt
