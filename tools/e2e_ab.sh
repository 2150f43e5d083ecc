#!/bin/bash
# A/B of the e2e (host-buffer) number between prebuilt libbsgd.so variants; run under gpurun.
tag=$1; shift
mkdir -p gpurun_out
cp paper_1903_11874_b200/libbsgd.so /tmp/libbsgd_orig.so
for so in "$@"; do
  cp "$so" paper_1903_11874_b200/libbsgd.so
  echo "== $so" >> gpurun_out/e2e_$tag.log
  python bench.py --steps 5 --warmup 3 --no-cpu --no-tv --cheap-data 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" >> gpurun_out/e2e_$tag.log 2>&1
done
cp /tmp/libbsgd_orig.so paper_1903_11874_b200/libbsgd.so
