# one GPU session: tests, smoke, bench, launch list + full ncu capture of k_simulate
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
for sh in 1 8; do python tools/profile_sweep.py --shards $sh --launches 2; done > gpurun_out/shards.log 2>&1
if [ -n "${NCU:-}" ]; then
python tools/profile_sweep.py --launches 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_simulate -c 1 -o gpurun_out/prof_sim -f python tools/profile_sweep.py --launches 1 > gpurun_out/ncu_full.log 2>&1
fi
for f in gpurun_out/*.log; do echo "== $f"; tail -4 $f; done
