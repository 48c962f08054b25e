#!/bin/bash
# K1+K2 micro-timings over library variants: bash scripts/hist_ab.sh "" _v1 ...
export VOXB200_NO_BUILD=1
for v in "$@"; do echo "== lib$v"; VOXB200_LIB=$PWD/paper_1807_03119_b200/libvoxb200$v.so python scripts/hist_micro.py 256 512 1024 2048 | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items(): print(k, v)"; done
