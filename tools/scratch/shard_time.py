"""Kernel times of shard 0 of the C5 sweep split n ways, on one GPU (the
per-GPU critical path of strong scaling).  python tools/scratch/shard_time.py [n ...]"""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2511_21669_b200 import Simulator  # noqa: E402

path = os.environ.get("SPEC", "configs/c5_sweep_65536.yaml")
spec = open(path).read()
with Simulator(0) as s:
    for n in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
        nrep, _ = s.prepare_sweep(spec, base_dir=os.path.dirname(path), shard=0, n_shards=n)
        t = []
        for k in range(4):
            s.launch()
            s.sync()
            t.append(s.last_kernel_ms())
        sm = s.summaries()
        print(f"shards {n} replicas {nrep} events {int(sm['events_processed'].sum())} "
              f"sim {min(x['sim_ms'] for x in t[1:]):.2f} ms gen {min(x['stage_ms'] for x in t[1:]):.2f} ms", flush=True)
