#!/bin/bash
# Build the production library and its bounds-checked test variant in parallel
# (both must be current before a gpurun: the box does not rebuild).
cd "$(dirname "$0")/.."
python -m paper_1807_03119_b200._build > /tmp/vx_build.log 2>&1 &
p1=$!
python -m paper_1807_03119_b200._build --checked > /tmp/vx_build_checked.log 2>&1 &
p2=$!
wait $p1; r1=$?
wait $p2; r2=$?
tail -1 /tmp/vx_build.log; tail -1 /tmp/vx_build_checked.log
exit $((r1 | r2))
