"""Host phase timings of dsd_run_sweep (DSD_HOST_TIMING) on the C5 sweep:
  python tools/scratch/e2e_probe.py [n_devices]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
os.environ["DSD_HOST_TIMING"] = "1"
from paper_2511_21669_b200 import Simulator  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = Simulator(list(range(nd)) if nd > 1 else 0)
spec = open("configs/c5_sweep_65536.yaml").read()
for k in range(4):
    t = time.perf_counter()
    out = s.run_sweep(spec, base_dir="configs")
    print("e2e %.1f ms" % ((time.perf_counter() - t) * 1e3), file=sys.stderr, flush=True)
