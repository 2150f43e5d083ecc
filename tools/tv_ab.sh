# A/B of TV prox variants at 1024^3 (8 slabs); run under gpurun.  usage: tools/tv_ab.sh TAG "ENV" ...
tag=$1; shift
mkdir -p gpurun_out
for e in "$@"; do
  echo "== $e $(env $e python tools/tv_profile.py 1024 1024 1024 8 2>&1 | tail -1)" >> gpurun_out/tv_ab_$tag.log
done
