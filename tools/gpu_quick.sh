# quick GPU check: C5 timing (A/B against build/ab/base.so when present), the
# lone-warp gamma=1 subset, then the GPU parity suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
  if [ -f build/ab/base.so ]; then echo -n "base "; DSD_LIB=$PWD/build/ab/base.so python tools/profile_sweep.py --launches 3 2>&1 | tail -2 | head -1; fi
  echo -n "cur  "; python tools/profile_sweep.py --launches 3 2>&1 | tail -2 | head -1
done
if [ -f configs/sweeps/sub_g1.yaml ]; then echo -n "lone g1 "; python tools/profile_sweep.py --spec configs/sweeps/sub_g1.yaml --launches 2 2>&1 | tail -2 | head -1; fi
if [ -n "${PYTEST_K:-}" ]; then python -m pytest tests -q -x -m gpu -k "$PYTEST_K" 2>&1 | tail -3; else python -m pytest tests -q -x -m gpu 2>&1 | tail -3; fi
