#!/bin/bash
# Round-end measurement on one GPU (run under gpurun): the default bench line,
# the ncu launch list of the bench command and a --set full capture of one
# C3 view's kernels.  Each ncu pass runs only after the same command exited 0
# without ncu.  Usage: tools/profile_round.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.log || exit 1
tail -1 gpurun_out/bench_$tag.json
cmd="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
$cmd > gpurun_out/pre_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
      --log-file gpurun_out/launches_$tag.csv $cmd > gpurun_out/ncu_launch_$tag.log 2>&1
echo "launch list rc=$?"
cmd1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
SGTR_LANES=1 $cmd1 > gpurun_out/pre1_$tag.log 2>&1 && \
  SGTR_LANES=1 ncu --set full --import-source on --clock-control none --kernel-name-base function \
      -k regex:"^(k_raster_vjp_wide|k_raster_fwd_bits|k_chain_warp|k_ssim|k_gather|k_project|k_tile_ids|k_emit_small)$" \
      -s 700 -c 10 -o gpurun_out/prof_full_$tag $cmd1 > gpurun_out/ncu_full_$tag.log 2>&1
echo "full capture rc=$?"
