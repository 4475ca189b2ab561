# A/B of kernel builds on sweep specs: for each spec, each library ($LIBS), 2 runs
cd $GRAFT_REPO_ROOT
for spec in ${SPECS:-configs/sweeps/dyn_8k.yaml}; do
  for i in 1 2; do
    for L in ${LIBS:-paper_2511_21669_b200/libdsdsim.so}; do
      echo -n "$(basename $L) $(basename $spec) "; DSD_LIB=$PWD/$L python tools/profile_sweep.py --spec $spec --launches 3 2>&1 | tail -2 | head -1 | sed 's/.*sim_ms/sim_ms/'
    done
  done
done
