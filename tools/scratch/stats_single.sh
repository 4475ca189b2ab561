# step statistics of the large-topology single runs, solo mode off / on
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
G=tests/golden/configs; X=tests/golden/_gen
for solo in ${SOLOS:-0 1}; do
  for c in "$G/c2_8x1_batching.yaml $G" "$G/c3_64x4_awc.yaml $X" "$G/c4_1024x16_static.yaml $X"; do
    echo "== solo=$solo $c"
    DSD_SOLO=$solo DSD_STEP_STATS=1 DSD_HOST_TIMING=1 python tools/scratch/run_one.py $c 2>&1 | grep -v "^\[dsd host\]" | tail -30
  done
done > gpurun_out/stats_single_${TAG:-x}.txt 2>&1
