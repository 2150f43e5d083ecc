#!/bin/bash
# Run on the GPU box (via gpurun): launch list of this library's kernels + one full
# ncu capture of the FP and BP launches of a cfg5 bench epoch.  Output: gpurun_out/.
# The bench's data generation (torch) is not profiled: kernels are filtered by name.
set -x
TAG=${1:-r01}
KSEL='regex:k_(project|residual|block_update|zero_rows|obj|axpy|dot3)'
mkdir -p gpurun_out
# every launch of ours with its device time (cold-cache, serialised: compare SHARES only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$KSEL" \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --cheap-data > gpurun_out/launches_${TAG}.log 2>&1
# the projector kernels, once each (FP then BP of the timed epoch)
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:k_project -s 2 -c 2 -o gpurun_out/prof_${TAG} -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --cheap-data > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
