# 2 or 4 GPUs: multi-rank parity + bench with the peer-memory transport and with NCCL (PIC_P2P=0).
mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
for mode in 1 0; do
  for n in 32 64; do
    MP_EXPECT_TRANSPORT=$([ $mode = 1 ] && echo peer || echo nccl) PIC_P2P=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port $((29700+n+mode)) tests/mp_worker.py $n 8 20 > gpurun_out/mp_P${NG}_n${n}_p2p$mode.log 2>&1
    echo "p2p=$mode mp P=$NG n=$n rc=$?"; grep -E "MP OK|Error|error|Traceback" gpurun_out/mp_P${NG}_n${n}_p2p$mode.log | head -3
  done
done
for mode in 1 0; do
  PIC_P2P=$mode timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29802+mode)) bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scale_P${NG}_p2p$mode.json 2> gpurun_out/scale_P${NG}_p2p$mode.err; echo "p2p=$mode bench P=$NG rc=$?"
  tail -1 gpurun_out/scale_P${NG}_p2p$mode.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], '%.3e'%d['value']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items()]" 2>&1 | head -16
  tail -3 gpurun_out/scale_P${NG}_p2p$mode.err
done
