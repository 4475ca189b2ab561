"""generate_dataset on the default DatasetGrid (200 scenarios x 12 candidates,
`specsim gen-dataset`): the GPU engine vs the reference library on all host cores."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import reforacle as ref  # noqa: E402
from paper_2511_21669_b200 import Simulator  # noqa: E402

with Simulator(0) as s:
    s.generate_dataset("")  # warm
    t = time.perf_counter()
    ds, _ = s.generate_dataset("")
    g = time.perf_counter() - t
t = time.perf_counter()
rds, _ = ref.generate_dataset("")
r = time.perf_counter() - t
print(f"generate_dataset default grid: gpu {g * 1e3:.0f} ms, reference {r * 1e3:.0f} ms "
      f"({os.cpu_count()} host threads), identical: {ds == rds}")
