# solo mode on / off over the large-topology workloads
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for solo in ${SOLOS:-1 0}; do
  DSD_SOLO=$solo WORKLOADS="${WL:-c2_single c3_single c4s_single c2_seeds c3_seeds}" TAG=solo$solo bash tools/workloads.sh 2>&1 | tail -8
done
