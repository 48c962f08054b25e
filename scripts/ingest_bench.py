"""§8f2 ingestion timing: load_raw of a u16 CT file straight to the device vs
the reference's host path (np.fromfile + FP64 rescale, volume.py:144-150),
and load_slice_stack of 8-bit PGM slices.  Page cache warm (file just
written); prints one JSON object."""
import json, os, sys, tempfile, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200.images import write_pgm

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tmp = tempfile.mkdtemp(dir=os.environ.get("INGEST_DIR", "/tmp"))
rs = np.random.default_rng(0)
n = edge ** 3
wide = rs.integers(0, 65536, n, dtype=np.uint16)
path = os.path.join(tmp, "ct.raw")
wide.tofile(path)
meta = vx.VolumeMeta(dims=(edge,) * 3, bit_depth=16)
res = {"edge": edge, "file_bytes": 2 * n}
vx.load_raw(path, meta)  # warm (library, pools)
t0 = time.perf_counter()
v = vx.load_raw(path, meta)
dt = time.perf_counter() - t0
res["load_raw_u16_s"] = dt
res["load_raw_u16_GBps_file"] = 2 * n / dt / 1e9
if edge <= 512:
    t0 = time.perf_counter()
    raw = np.fromfile(path, dtype="<u2")
    ref = np.floor(raw.astype(np.float64) * 255.0 / 65535.0 + 0.5).astype(np.uint8)
    res["reference_host_rescale_s"] = time.perf_counter() - t0
    assert np.array_equal(ref, v.data.reshape(-1))
del v
os.remove(path)
# slice stack: edge slices of edge x edge
sl_dir = os.path.join(tmp, "slices")
os.mkdir(sl_dir)
planes = rs.integers(0, 256, (min(edge, 512), edge, edge), dtype=np.uint8)
for i, p in enumerate(planes):
    write_pgm(p, os.path.join(sl_dir, f"s{i:04d}.pgm"))
vx.load_slice_stack(sl_dir)
t0 = time.perf_counter()
v = vx.load_slice_stack(sl_dir)
dt = time.perf_counter() - t0
res["slices"] = [int(x) for x in planes.shape]
res["load_slice_stack_s"] = dt
res["load_slice_stack_GBps"] = planes.size / dt / 1e9
assert np.array_equal(v.data, planes)
print(json.dumps(res))
