# one GPU session: smoke, GPU parity tests, bench, shard timings, and (NCU=1)
# the launch list of a short bench run + one full ncu capture of k_simulate
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
for sh in 1 8; do python tools/profile_sweep.py --shards $sh --launches 2; done > gpurun_out/shards.log 2>&1
if [ -n "${NCU:-}" ]; then
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
  python tools/profile_sweep.py --launches 1 > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_simulate -c 1 -o gpurun_out/prof_sim -f \
      python tools/profile_sweep.py --launches 1 > gpurun_out/ncu_full.log 2>&1
fi
for f in gpurun_out/*.log; do echo "== $f"; tail -4 $f; done
