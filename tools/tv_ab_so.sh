#!/bin/bash
# A/B of TV prox kernels between prebuilt libbsgd.so variants at 1024^3 (8 slabs); run under gpurun.
# usage: tools/tv_ab_so.sh TAG "ENV" variants/a.so variants/b.so ...
tag=$1; env_=$2; shift 2
mkdir -p gpurun_out
cp paper_1903_11874_b200/libbsgd.so /tmp/libbsgd_orig.so
for so in "$@"; do
  cp "$so" paper_1903_11874_b200/libbsgd.so
  echo "== $so $env_ $(env $env_ python tools/tv_profile.py 1024 1024 1024 8 2>&1 | tail -1)" >> gpurun_out/tv_ab_$tag.log
done
cp /tmp/libbsgd_orig.so paper_1903_11874_b200/libbsgd.so
