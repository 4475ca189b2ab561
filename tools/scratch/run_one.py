"""Runs one config once through dsd_run_simulation (for ncu captures).
  python tools/run_one.py <config.yaml> [base_dir]"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2511_21669_b200 import Simulator  # noqa: E402

cfg = sys.argv[1]
base = sys.argv[2] if len(sys.argv) > 2 else os.path.dirname(os.path.abspath(cfg))
with Simulator(0) as s:
    out = s.run_simulation(open(cfg).read(), base_dir=base)
    print("events", out.events_processed)
