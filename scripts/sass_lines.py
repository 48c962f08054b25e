"""Attribute ncu per-SASS stall samples / executed instructions to source lines.

    python scripts/sass_lines.py <sass.csv from ncu --page source --print-source sass>
        <nvdisasm -g -c dump> <kernel mangled-name substring> [top]
"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dump, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
iA, iS, iI = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
    "Instructions Executed")
samples = {}
for r in rows[2:]:
    samples[int(r[iA], 16)] = (float(r[iS] or 0), float(r[iI] or 0))
base = min(samples)
line_of = {}
cur = None
inside = False
for l in open(dump):
    if l.startswith("//----") and ".text." in l:
        inside = kname in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0.0, 0.0])
for a, (s, i) in samples.items():
    ln = line_of.get(a - base)
    agg[ln][0] += s
    agg[ln][1] += i
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
srcs = {}


def text_of(key):
    if not key:
        return "?", "?"
    f, ln = key
    if f not in srcs:
        try:
            srcs[f] = open(f).read().splitlines()
        except OSError:
            srcs[f] = []
    src = srcs[f]
    name = f"{f.rsplit('/', 1)[-1]}:{ln}"
    return name, (src[ln - 1].strip()[:80] if ln <= len(src) else "?")


for key, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    name, text = text_of(key)
    print(f"{name:>28} stall {100*s/ts:5.1f}% inst {100*i/ti:5.1f}%  {text}")
