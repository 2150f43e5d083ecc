#!/bin/bash
# Run on the GPU box (via gpurun): launch list of this library's kernels + ncu captures of the
# FP and BP launches of a timed cfg5 bench epoch, one block update and one TV iteration.
# Output: gpurun_out/.  k_project3 launch order in `bench.py --warmup 1 --steps 1`: 4 COUNT
# launches (visit table, one per detector tile), warm-up FP, BP, timed FP, BP -> skip 6.
set -x
TAG=${1:-r02}
KSEL='regex:k_(project|residual|normsq_final|block_update|zero_rows|obj|axpy|dot3|tv_)'
mkdir -p gpurun_out
# every launch of ours with its device time (cold-cache, serialised: compare SHARES only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$KSEL" \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-tv --cheap-data > gpurun_out/launches_${TAG}.log 2>&1
# FP: the full set with source counters
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_project3 -s 6 -c 1 -o gpurun_out/prof_fp_${TAG} -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-tv --cheap-data > gpurun_out/prof_fp_${TAG}.log 2>&1
# BP: the sections that replay reliably with the atomics
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis \
  --section WarpStateStats --section SchedulerStats --section Occupancy --section LaunchStats \
  --metrics lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
  --clock-control none -k regex:k_project3 -s 7 -c 1 -o gpurun_out/prof_bp_${TAG} -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-tv --cheap-data > gpurun_out/prof_bp_${TAG}.log 2>&1
# one block update (a slab) and one two-iteration TV pass (k_tv_fgp_z2, the one-rank default)
timeout 600 ncu --set full --clock-control none -k regex:k_block_update -s 8 -c 1 -o gpurun_out/prof_upd_${TAG} -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-tv --cheap-data > gpurun_out/prof_upd_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_tv_fgp_z2 -s 14 -c 1 -o gpurun_out/prof_tv_${TAG} -f \
  python tools/tv_profile.py 1024 1024 1024 8 > gpurun_out/prof_tv_${TAG}.log 2>&1
ls -la gpurun_out
