import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["DSD_HOST_TIMING"] = "1"
from paper_2511_21669_b200 import Simulator
s = Simulator(0)
spec = open("configs/c5_sweep_65536.yaml").read()
for k in range(3):
    t = time.perf_counter()
    out = s.run_sweep(spec, base_dir="configs")
    print("e2e %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
