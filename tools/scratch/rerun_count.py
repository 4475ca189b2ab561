"""How many replicas of a sweep the shared-memory kernel hands to the HBM
variant (heap or specialised-stack overflow): python tools/rerun_count.py spec.yaml..."""
import os
import sys

os.environ["DSD_HOST_TIMING"] = "1"
sys.path.insert(0, os.getcwd())
from paper_2511_21669_b200 import Simulator  # noqa: E402

with Simulator(0) as s:
    for spec in sys.argv[1:]:
        print("==", spec, flush=True)
        s.prepare_sweep(spec)
        s.launch()
        s.sync()
