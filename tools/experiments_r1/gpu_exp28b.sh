OUT=gpurun_out/exp28b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for T in synccheck; do
  timeout 1200 compute-sanitizer --tool $T python tools/sanitize_cases.py > $OUT/san_$T.txt 2>&1
  echo "rc=$?" >> $OUT/san_$T.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or star or randomised or epoch" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
