set -x
timeout 600 python -m pytest tests/test_gpu_stats.py tests/test_gpu_large.py -q -x --timeout 500 -p no:cacheprovider > gpurun_out/pt2.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pt2.log
timeout 300 python scripts/config_sweep.py --hist-only > gpurun_out/hist_sweep.json 2> gpurun_out/hist_sweep.err; echo sweep rc=$?
timeout 300 python scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; echo e2e rc=$?
cat gpurun_out/e2e_breakdown.txt
python -c "
import json;d=json.load(open('gpurun_out/hist_sweep.json'));print(json.dumps(d['C5_hist_sweep']))"
