# A/B of the cooperative first-candidate variants (frames + bench + GPU tests on one variant)
set -x
bash scripts/ab_sweep.sh "" ${VARIANTS:-_pair2 _pair4 _pair6} > gpurun_out/ab.txt 2>&1
for v in "" ${VARIANTS:-_pair2 _pair4 _pair6}; do
  VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200$v.so VOXB200_NO_BUILD=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench$v.json 2>/dev/null
done
VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200${TESTV:-_pair6}.so VOXB200_NO_BUILD=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_variant.log 2>&1; echo pytest rc=$?
