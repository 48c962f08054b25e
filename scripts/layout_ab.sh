#!/bin/bash
# Voxel-layout A/B: the linear apron replica vs 8^3 bricks
# (linear inside / Morton inside) for K4's reads.  Parity of each variant,
# frame times over the configs, the no-skip (full traversal) leg, and one ncu
# metric pass per variant over the bench frame (K4: DRAM bytes, L1 sectors
# per request, L1/L2 hit rates, issue activity).
#   bash scripts/layout_ab.sh "" _brick1 _brick2
set -u
mkdir -p gpurun_out
export VOXB200_NO_BUILD=1
for v in "$@"; do
  export VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200$v.so
  echo "== lib$v"
  timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_render.py \
    "tests/test_gpu_large.py::test_bench_frame_1024_full_vs_oracle" > gpurun_out/layout_tests$v.log 2>&1
  echo "tests rc=$? $(tail -1 gpurun_out/layout_tests$v.log)"
  timeout 600 python bench.py --steps 20 --warmup 5 --ncu off --no-cpu --orbit 0 --noskip-steps 5 \
    > gpurun_out/layout_bench$v.log 2>&1
  echo "bench rc=$?"
done
unset VOXB200_LIB
SWEEP_TIMEOUT=300 bash scripts/ab_sweep.sh "$@"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for v in "$@"; do
  VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200$v.so timeout 600 ncu --metrics $M --clock-control none \
    -k regex:raycast_kernel -c 4 --csv --log-file gpurun_out/ncu_layout$v.csv \
    python bench.py --ncu-child > gpurun_out/ncu_layout$v.out 2>&1
  echo "ncu$v rc=$?"
done
