#!/bin/bash
# compute-sanitizer over scripts/sanitize_target.py with ONE tool (run one
# tool per gpurun call: several tools in one call have hung B200 boxes,
# /opt/skills/guides/B200_PROFILING.md).  Usage: scripts/sanitize.sh memcheck
set -uo pipefail
TOOL=${1:?tool: memcheck|racecheck|synccheck|initcheck}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export VOXB200_NO_BUILD=1
python scripts/sanitize_target.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
EXTRA=""
[ "$TOOL" = memcheck ] && EXTRA="--leak-check no"
[ "$TOOL" = racecheck ] && EXTRA="--racecheck-report all"
timeout 1500 compute-sanitizer --tool "$TOOL" $EXTRA --error-exitcode 9 --print-limit 50 \
    python scripts/sanitize_target.py > "gpurun_out/sanitize_$TOOL.log" 2>&1
rc=$?
echo "compute-sanitizer --tool $TOOL rc=$rc"
tail -8 "gpurun_out/sanitize_$TOOL.log"
exit $rc
