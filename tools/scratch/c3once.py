import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import reforacle as ref
from paper_2511_21669_b200 import Simulator
with Simulator(0) as s:
    text = open(os.path.join(ref.CONFIGS, "c3_64x4_awc.yaml")).read()
    s.run_simulation(text, base_dir=ref.GEN_DIR)
    t = time.perf_counter(); out = s.run_simulation(text, base_dir=ref.GEN_DIR); print("c3 %.1f ms" % ((time.perf_counter() - t) * 1e3), os.environ.get("DSD_AWC_CARVEOUT"))
