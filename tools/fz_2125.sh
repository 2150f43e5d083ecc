for so in variants/fine13.so variants/cur.so variants/final.so variants/base.so; do
  cp $so paper_1903_11874_b200/libbsgd.so
  echo "== $so" >> gpurun_out/s33_fz.log
  timeout 300 python tools/fuzz_sweep.py 2125 2126 operator 2>&1 | grep -E "AssertionError|fuzz seeds" >> gpurun_out/s33_fz.log
done
cp variants/fine13.so paper_1903_11874_b200/libbsgd.so
timeout 300 python tests/debug_fuzz.py 2125 17 > gpurun_out/s33_dbg.log 2>&1
