timeout 300 python -m pytest tests/test_gpu_stats.py -q -x -p no:cacheprovider > gpurun_out/pt_stats.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pt_stats.log)"
timeout 300 python scripts/hist_micro.py 256 512 1024 > gpurun_out/hist_micro.json 2>&1; cat gpurun_out/hist_micro.json | tr -d '\n '; echo
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hist --csv python scripts/hist_micro.py 256 512 1024 > gpurun_out/hist_ncu.csv 2>&1; echo ncu rc=$?
