# The gamma=1 subset (round 1's critical path): step statistics, the
# per-replica cost table, one ncu --set full capture; the AWC sweep vs the
# reference's run_sweep on every host core
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DSD_STEP_STATS=1 python tools/profile_sweep.py --spec configs/sweeps/sub_g1.yaml --launches 1 > gpurun_out/hv_stats.txt 2>&1
python tools/profile_sweep.py --spec configs/sweeps/sub_g1.yaml --launches 3 > gpurun_out/hv_plain.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_simulate -c 1 -o gpurun_out/hv_full -f \
    python tools/profile_sweep.py --spec configs/sweeps/sub_g1.yaml --launches 1 > gpurun_out/hv_ncu.log 2>&1
python - > gpurun_out/awc_vs_ref.json 2>&1 <<'PY'
import json, os, sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import reforacle as ref
from paper_2511_21669_b200 import Simulator
spec = open("configs/sweeps/awc_sweep.yaml").read()
base = "configs/sweeps"
with Simulator(0) as s:
    s.run_sweep(spec, base_dir=base)
    t = time.perf_counter(); out = s.run_sweep(spec, base_dir=base); g = time.perf_counter() - t
r = ref.sweep_bench(spec, base, os.cpu_count())
print(json.dumps({"workload": "configs/sweeps/awc_sweep.yaml: 48 points x 16 reps, single pair, AWC window",
                  "gpu_e2e_s": g, "events": out.events_processed, "gpu_events_per_s": out.events_processed / g,
                  "reference_s": r["seconds"], "reference_threads": os.cpu_count(),
                  "reference_events_per_s": r["events"] / r["seconds"], "ratio": r["seconds"] / g}))
PY
tail -3 gpurun_out/hv_plain.txt; cat gpurun_out/awc_vs_ref.json
