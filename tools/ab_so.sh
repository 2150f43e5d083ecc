# A/B of prebuilt libbsgd.so variants on the cfg5 bench (device time); run under gpurun.
# usage: tools/ab_so.sh TAG variants/a.so variants/b.so ...
tag=$1; shift
mkdir -p gpurun_out
cp paper_1903_11874_b200/libbsgd.so /tmp/libbsgd_orig.so
for so in "$@"; do
  cp "$so" paper_1903_11874_b200/libbsgd.so
  echo "== $so" >> gpurun_out/ab_$tag.log
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-tv --cheap-data 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phase_ms'], d['roofline']['fp_frac'], d['roofline']['bp_frac'])" >> gpurun_out/ab_$tag.log 2>&1
done
cp /tmp/libbsgd_orig.so paper_1903_11874_b200/libbsgd.so
