#!/bin/bash
# Round-2 profile set (one gpurun call; ncu wrapper runs each command plain first):
#  1. full ncu capture of the warm skipping K4 of the bench frame
#  2. K4 memory/issue metrics of C3 sigma and entropy frames (staging question)
#  3. launch list of a short bench run
set -u
mkdir -p gpurun_out
export VOXB200_NO_BUILD=1
ncu --set full --clock-control none --import-source on -k regex:raycast_kernel -s 2 -c 1 \
    -o gpurun_out/k4_full -f python bench.py --ncu-child > gpurun_out/k4_full.out 2>&1
echo "full rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio
for k in sigma entropy local-cluster; do
  ncu --metrics $M --clock-control none -k regex:raycast_kernel -c 4 --csv \
      --log-file gpurun_out/ncu_c3_$k.csv python scripts/render_once.py 512 $k > gpurun_out/ncu_c3_$k.out 2>&1
  echo "c3 $k rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --ncu off --no-cpu --orbit 0 --noskip-steps 0 --no-e2e > gpurun_out/bench_launches.out 2>&1
echo "launches rc=$?"
