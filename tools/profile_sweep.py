"""Runs the C5 sweep's kernels a few times (for ncu captures): prepare once,
then `--launches` launches of the staging + simulation kernels."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_21669_b200 import Simulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--spec", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                               "configs", "c5_sweep_65536.yaml"))
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--shard", type=int, default=0)
ap.add_argument("--shards", type=int, default=1)
a = ap.parse_args()
s = Simulator(0)
n, p = s.prepare_sweep(a.spec, shard=a.shard, n_shards=a.shards)
for _ in range(a.launches):
    s.launch()
    s.sync()
    print(n, p, s.last_kernel_ms(), flush=True)
sm = s.summaries()
print("events", int(sm["events_processed"].sum()), "failed", int((sm["status"] != 0).sum()))
