# A/B of library builds ($LIBS) on the C5 shard times (tools/scratch/shard_time.py), $ROUNDS rounds
cd $GRAFT_REPO_ROOT
for i in $(seq ${ROUNDS:-2}); do
  for L in ${LIBS:-build/ab/base.so paper_2511_21669_b200/libdsdsim.so}; do
    echo "== $(basename $L)"; DSD_LIB=$PWD/$L python tools/scratch/shard_time.py ${SHARDS:-1 2 4 8} 2>&1 | grep shards
  done
done
