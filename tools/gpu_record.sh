# One recording session (gpurun --gpus 4): bench lines at N=1,2,4 (strong
# scaling), the reference arm, the ncu launch list of the bench command and
# one ncu --set full capture of k_simulate; outputs in gpurun_out/rec_*
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/rec
python bench.py --steps 10 --warmup 3 > ${O}_n1.json 2> ${O}_n1.err
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
    bench.py --gpus $n --steps 10 --warmup 3 > ${O}_n$n.json 2> ${O}_n$n.err
done
python bench.py --impl reference --steps 2 --warmup 3 > ${O}_ref.json 2> ${O}_ref.err
python tools/profile_sweep.py --launches 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > ${O}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_simulate -c 1 -o ${O}_full -f \
    python tools/profile_sweep.py --launches 1 > ${O}_ncu_full.log 2>&1
for f in ${O}_n1.json ${O}_n2.json ${O}_n4.json ${O}_ref.json; do echo "== $f"; cut -c1-400 $f; done
