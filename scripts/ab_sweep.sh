#!/bin/bash
# A/B the frame configs over library variants in one box session:
#   bash scripts/ab_sweep.sh "" _variant ...   ("" = the default library)
mkdir -p gpurun_out
for v in "$@"; do
  echo "== lib$v"
  VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200$v.so VOXB200_NO_BUILD=1 timeout ${SWEEP_TIMEOUT:-180} \
    python scripts/config_sweep.py --frames-only --reps 20 > gpurun_out/sweep$v.json 2>gpurun_out/sweep$v.err
  python - "$v" <<'PY'
import json, sys
r = json.load(open(f"gpurun_out/sweep{sys.argv[1]}.json"))
for k, v in r.items():
    if isinstance(v, dict) and "filters" in v:
        print(k, {f: round(x["ms"], 4) for f, x in v["filters"].items()})
PY
done
