# One round's measurement set: bench line, reference arm, launch list, K4 + K1/K2 full captures, config sweep.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"raycast|tile_order|hist|otsu|dist_|accept|cell_max|brick_max|span_max|entropy" --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:raycast_kernel -s 8 -c 1 -o gpurun_out/raycast_full \
  python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > gpurun_out/ncu_k4.log 2>&1; echo k4 rc=$?
ncu --set full --clock-control none -k regex:hist_otsu -c 1 -o gpurun_out/hist_otsu_full \
  python scripts/hist_once.py > gpurun_out/ncu_hist.log 2>&1; echo hist rc=$?
timeout 600 python scripts/config_sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo sweep rc=$?
python scripts/cold_frames.py > gpurun_out/cold.txt 2>&1; echo cold rc=$?
