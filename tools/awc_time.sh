# AWC timings (C3 / C4-awc single runs, the 768-replica AWC sweep, the AWC
# dataset) for the current build and the libraries in $ALT_LIBS
cd $GRAFT_REPO_ROOT
for L in ${ALT_LIBS:-} paper_2511_21669_b200/libdsdsim.so; do
  echo "== $L"
  for w in c3_single c4a_single; do
    DSD_LIB=$PWD/$L python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],1), 'ms')"
  done
  DSD_LIB=$PWD/$L python tools/profile_sweep.py --spec configs/sweeps/awc_sweep.yaml --launches 2 2>&1 | tail -2 | head -1
  DSD_LIB=$PWD/$L python tools/dataset_time.py 2>&1 | tail -1
done
