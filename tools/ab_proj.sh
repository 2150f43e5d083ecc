#!/bin/bash
# A/B of projector variants on the cfg5 bench (device time only); run under gpurun.
# usage: tools/ab_proj.sh TAG "ENV1" "ENV2" ...   (each ENV: space-separated VAR=value list)
tag=$1; shift
mkdir -p gpurun_out
for e in "$@"; do
  echo "== $e" >> gpurun_out/ab_$tag.log
  env $e python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-tv --cheap-data 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phase_ms'], d['roofline']['fp_frac'], d['roofline']['bp_frac'])" >> gpurun_out/ab_$tag.log 2>&1
done
