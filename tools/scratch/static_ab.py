import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import reforacle as ref
from paper_2511_21669_b200 import Simulator
gen = ref.GEN_DIR
with Simulator(0) as s:
    for name in ["c1_single_pair.yaml", "c2_8x1_batching.yaml", "c4_1024x16_static.yaml"]:
        text = open(os.path.join(ref.CONFIGS, name)).read()
        s.run_simulation(text, base_dir=gen)
        ts = []
        for _ in range(3):
            t = time.perf_counter(); s.run_simulation(text, base_dir=gen); ts.append(time.perf_counter() - t)
        print(os.environ.get("DSD_LIB", "cur")[-10:], name, "%.1f ms" % (1e3 * min(ts)), flush=True)
