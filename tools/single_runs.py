"""Times single-replica runs through dsd_run_simulation on
the GPU and through the reference library on one host core."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import reforacle as ref  # noqa: E402
from paper_2511_21669_b200 import Simulator  # noqa: E402

ref.ensure_generated()
gen = ref.GEN_DIR
with Simulator(0) as s:
    for name in ["c1_single_pair.yaml", "c2_8x1_batching.yaml", "c3_64x4_awc.yaml", "c4_1024x16_static.yaml",
                 "c4_1024x16_awc.yaml"]:
        text = open(os.path.join(ref.CONFIGS, name)).read()
        s.run_simulation(text, base_dir=gen)  # warm
        t = time.perf_counter()
        out = s.run_simulation(text, base_dir=gen)
        g = time.perf_counter() - t
        t = time.perf_counter()
        rep, ev, end, agg = ref.run_config(text, gen, None)
        c = time.perf_counter() - t
        assert ev == out.events_processed
        print(f"{name:24s} events {ev:9d}  gpu {g * 1e3:9.1f} ms  ref-cpu(1 core) {c * 1e3:9.1f} ms", flush=True)
