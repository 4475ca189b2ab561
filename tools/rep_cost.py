"""Per-replica cost of a sweep (lane placement / sharding cost model).

Runs the sweep once with DSD_STEP_STATS=1 and DSD_REP_STATS_FILE (a build with
-DDSD_REP_STATS, e.g. DSD_LIB=build/ab/repstats.so, also counts session-loop
iterations) and prints, per value of each axis, the mean vote rounds, loop
iterations, events and cycles of its replicas; then a least-squares fit
cycles ~ A * requests + B * iterations + C * rounds.

  DSD_LANES_PER_WARP=1 DSD_LIB=build/ab/repstats.so python tools/rep_cost.py [spec] [--shards=N]
"""
import collections
import ctypes
import os
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
args = [a for a in sys.argv[1:] if not a.startswith("--shards=")]
shards = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--shards=")), 1))
spec_path = args[0] if args else os.path.join(REPO, "configs", "c5_sweep_65536.yaml")
out = tempfile.mktemp()
os.environ["DSD_STEP_STATS"] = "1"
os.environ["DSD_REP_STATS_FILE"] = out
from paper_2511_21669_b200 import Simulator, _lib  # noqa: E402

L = _lib.lib()
text = open(spec_path).read()
base = os.path.dirname(os.path.abspath(spec_path))
p = ctypes.c_void_p()
err = ctypes.create_string_buffer(1024)
assert L.dsd_plan_sweep(text.encode(), base.encode(), 0, shards, ctypes.byref(p), err, 1024) == 0, err.value
n = L.dsd_sweep_plan_replicas(p, None)
pts = (ctypes.c_int64 * n)()
L.dsd_sweep_plan_origin(p, pts, None, n)
s = Simulator(0)
s.prepare_sweep(text, base_dir=base, shard=0, n_shards=shards)
s.launch()
s.sync()
sm = s.summaries()
rs = np.fromfile(out, dtype=np.uint64).reshape(-1, 3).astype(np.float64)
os.unlink(out)
# axes from the spec text (values in declaration order; point index is mixed radix, last axis fastest)
axes = []
for line in text.splitlines():
    line = line.strip()
    if ":" in line and "[" in line:
        k, v = line.split(":", 1)
        axes.append((k.strip(), [x.strip() for x in v.strip().strip("[]").split(",")]))
pt = np.array(list(pts), dtype=np.int64)
idx = {}
rem = pt.copy()
for k, vals in reversed(axes):
    idx[k] = rem % len(vals)
    rem //= len(vals)
axes_v = dict(axes)
ev = sm["events_processed"].astype(np.float64)
req = sm["n_requests"].astype(np.float64)
for k, vals in axes:
    print(f"== {k}")
    for j, v in enumerate(vals):
        m = idx[k] == j
        print(f"  {v:>6}: rounds {rs[m, 0].mean():8.0f}  iters {rs[m, 1].mean():8.0f}  events {ev[m].mean():8.0f}"
              f"  Mcycles {rs[m, 2].mean() / 1e6:7.3f}")
print("== the 16 most expensive replicas (Mcycles; shard 0 of %d)" % shards)
for r in np.argsort(-rs[:, 2])[:16]:
    print("  " + "  ".join(f"{k.split('.')[-1]}={axes_v[k][idx[k][r]]}" for k in axes_v) +
          f"  events {ev[r]:8.0f} requests {req[r]:5.0f} rounds {rs[r, 0]:8.0f} Mcycles {rs[r, 2] / 1e6:7.3f}")
X = np.stack([req, rs[:, 1], rs[:, 0]], axis=1)
coef, *_ = np.linalg.lstsq(X, rs[:, 2], rcond=None)
pred = X @ coef
print("fit cycles ~ %.0f*requests + %.0f*iters + %.0f*rounds; rel.err mean %.3f" %
      (coef[0], coef[1], coef[2], np.mean(np.abs(pred - rs[:, 2]) / rs[:, 2])))
