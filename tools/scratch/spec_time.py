"""Kernel time of a sweep spec given inline (base dir configs/):
  python tools/scratch/spec_time.py 'gamma: [15]' 'acceptance_rate: [0.92]' ..."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2511_21669_b200 import Simulator  # noqa: E402

axes = {"policies.window.gamma": "[15]", "network.rtt_ms": "[2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30, 32]",
        "workload.acceptance_rate": "[0.92]"}
reps = 16
for a in sys.argv[1:]:
    k, v = a.split(":", 1)
    if k == "reps":
        reps = int(v)
        continue
    axes[next(x for x in axes if x.endswith(k))] = v.strip()
spec = f"base: c1_single_pair.yaml\nseed: 42\nrepetitions: {reps}\naxes:\n" + "".join(f"  {k}: {v}\n" for k, v in axes.items())
with Simulator(0) as s:
    nrep, _ = s.prepare_sweep(spec, base_dir="configs")
    t = []
    for k in range(3):
        s.launch()
        s.sync()
        t.append(s.last_kernel_ms())
    sm = s.summaries()
    print(" ".join(sys.argv[1:]), f"replicas {nrep} events/replica {sm['events_processed'].mean():.0f} max {sm['events_processed'].max()}"
          f" sim {min(x['sim_ms'] for x in t[1:]):.2f} ms", flush=True)
