for so in variants/cur.so variants/final.so variants/base.so; do
  cp $so paper_1903_11874_b200/libbsgd.so
  echo "== $so" >> gpurun_out/s31_fz.log
  timeout 300 python tools/fuzz_sweep.py 1598 1599 operator 2>&1 | grep -E "AssertionError|fuzz seeds" >> gpurun_out/s31_fz.log
done
cp variants/cur.so paper_1903_11874_b200/libbsgd.so
timeout 300 python tests/debug_fuzz.py 1598 158 > gpurun_out/s31_dbg.log 2>&1
