#!/bin/bash
# A/B library variants (scripts/build_variant.py) in one box session: parity
# tests on every variant, the config sweep, and the bench line (incl. the
# no-skip leg) per variant.   bash scripts/variant_ab.sh "" _v1 _v2 ...
set -u
mkdir -p gpurun_out
export VOXB200_NO_BUILD=1
for v in "$@"; do
  export VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200$v.so
  timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_render.py tests/test_gpu_filters.py tests/test_gpu_volume.py \
    "tests/test_gpu_large.py::test_bench_frame_1024_full_vs_oracle" > gpurun_out/ab_tests$v.log 2>&1
  echo "lib$v tests rc=$? $(tail -1 gpurun_out/ab_tests$v.log)"
  timeout 600 python bench.py --steps 30 --warmup 5 --ncu off --no-cpu --orbit 0 --noskip-steps 5 \
    > gpurun_out/ab_bench$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads([x for x in open(f"gpurun_out/ab_bench{v}.log") if x.startswith("{")][0])
print(f"lib{v} bench {d['value']:.0f} fps kernel {d['roofline']['kernel_ms']:.4f} ms, "
      f"no-skip {d['roofline']['noskip']['kernel_ms']:.3f} ms, e2e {d['e2e']['value']:.0f}")
PY
done
unset VOXB200_LIB
SWEEP_TIMEOUT=300 bash scripts/ab_sweep.sh "$@"
