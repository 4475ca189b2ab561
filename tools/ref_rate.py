"""Reference run_sweep worker rate (events/s) on a strided sample of a sweep's
points, all host threads: python tools/ref_rate.py <sweep.yaml> <base_dir> <points>"""
import os
import sys

sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import reforacle as ref  # noqa: E402

spec, base, npts = open(sys.argv[1]).read(), sys.argv[2], int(sys.argv[3])
r = ref.sweep_bench(spec, base, os.cpu_count(), list(range(0, 256, max(1, 256 // npts))))
print("ref events/s %.3g (%d threads, %d replicas)" % (r["events"] / r["seconds"], os.cpu_count(), r["replicas"]))
