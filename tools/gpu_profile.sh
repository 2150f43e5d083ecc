#!/bin/bash
# Run on the GPU box (via gpurun): launch list + one full ncu capture of the FP and BP
# kernels of the cfg5 bench step.  Results land in gpurun_out/.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
# every launch with its device time (cold-cache, serialised: compare SHARES only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_${TAG}.log 2>&1
# the projector kernels, once each (FP then BP of a timed epoch)
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:k_project -s 4 -c 2 -o gpurun_out/prof_${TAG} -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
