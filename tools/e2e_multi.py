"""Host-path phases of dsd_run_sweep on one and on several GPUs (DSD_HOST_TIMING=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DSD_HOST_TIMING"] = "1"
from paper_2511_21669_b200 import Simulator  # noqa: E402

spec = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs", "c5_sweep_65536.yaml")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for devs in ([0], list(range(n))):
    with Simulator(devs) as s:
        for k in range(3):
            t = time.perf_counter()
            s.run_sweep(spec)
            print(devs, "run_sweep ms", round(1e3 * (time.perf_counter() - t), 2), file=sys.stderr, flush=True)
