# Bench lines for the BASELINE configs besides C5 (bench.py --workload ...):
# single runs and multi-seed sweeps of C1-C4, each with its reference
# cpu_baseline, into gpurun_out/workloads_<tag>.jsonl
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/workloads_${TAG:-run}.jsonl
: > $out
for w in ${WORKLOADS:-c1_single c2_single c3_single c4s_single c4a_single c2_seeds c3_seeds c4s_seeds c4a_seeds}; do
  python bench.py --workload $w --steps ${STEPS:-3} --warmup 3 >> $out 2>> gpurun_out/workloads_${TAG:-run}.err || echo "{\"workload\": \"$w\", \"failed\": true}" >> $out
done
python - "$out" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    d = json.loads(line)
    if d.get("failed"):
        print(d); continue
    cb = d.get("cpu_baseline", {})
    print(f'{d["config"]["workload"][:60]:60s} gpu {d["value"]:.3e} e2e {d["e2e"]["value"]:.3e} ms {d["ms_per_step"]:8.2f}'
          f' | ref {cb.get("value", 0):.3e} ({cb.get("cores")} cores) x{d["e2e"]["value"] / max(cb.get("value", 1), 1):.1f}')
PY
