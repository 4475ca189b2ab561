# A/B timing on the GPU box (scratch helper): for each spec (C5, the lone
# gamma=1 subset, $EXTRA_SPECS) time base (build/ab/base.so), the libraries in
# $ALT_LIBS and the current build; then the GPU tests selected by $PYTEST_K
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in configs/c5_sweep_65536.yaml configs/sweeps/sub_g1.yaml ${EXTRA_SPECS:-}; do
  for i in 1 2; do
    for L in build/ab/base.so ${ALT_LIBS:-} paper_2511_21669_b200/libdsdsim.so; do
      [ -f $L ] || continue
      echo -n "$(basename $L) $(basename $spec) "; DSD_LIB=$PWD/$L python tools/profile_sweep.py --spec $spec --launches 3 2>&1 | tail -2 | head -1 | sed 's/.*sim_ms/sim_ms/'
    done
  done
done
python tools/profile_sweep.py --launches 1 2>&1 | tail -1
if [ -n "${PYTEST_K:-}" ]; then timeout 900 python -m pytest tests -q -x -m gpu -k "$PYTEST_K" 2>&1 | tail -5; fi
