"""The C5 sweep at more repetitions (default 64: 262,144 replicas, ~3.5e9
events) on one or more GPUs of one handle: summary JSON/CSV against the
reference's run_sweep, and the timing.
  python tools/scratch/big_sweep.py [repetitions] [devices]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import reforacle as ref  # noqa: E402
from paper_2511_21669_b200 import Simulator  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ndev = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = open("configs/c5_sweep_65536.yaml").read().replace("repetitions: 16", f"repetitions: {reps}")
with Simulator(list(range(ndev)) if ndev > 1 else 0) as s:
    t = time.perf_counter()
    out = s.run_sweep(spec, base_dir="configs")
    dt = time.perf_counter() - t
    print(f"replicas {out.replicas} events {out.events_processed} e2e {dt * 1e3:.1f} ms", flush=True)
    t = time.perf_counter()
    out = s.run_sweep(spec, base_dir="configs")
    print(f"second call e2e {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
t = time.perf_counter()
js, cs = ref.run_sweep(spec, "configs", os.cpu_count())
print(f"reference run_sweep {time.perf_counter() - t:.1f} s on {os.cpu_count()} threads", flush=True)
print("summary JSON identical:", out.summary_json == js, " CSV identical:", out.summary_csv == cs)
