# histogram variants: parity (stats tests) + micro timings per cluster size
for v in "" cl2 cl4 cl8; do
  if [ -n "$v" ]; then export VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200_$v.so; else unset VOXB200_LIB; fi
  timeout 300 python -m pytest tests/test_gpu_stats.py -q -x -p no:cacheprovider > gpurun_out/pt_$v.log 2>&1; echo "variant=$v pytest rc=$? $(tail -1 gpurun_out/pt_$v.log)"
  timeout 300 python scripts/hist_micro.py 256 512 1024 2048 > gpurun_out/hist_micro_$v.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/hist_micro_$v.json'))
for k,r in d.items(): print('$v',k,r)"
done
