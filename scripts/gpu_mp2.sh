# 2-GPU: multi-rank parity workers + the P=2 bench.
mkdir -p gpurun_out
for n in 32 64; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29700+n)) tests/mp_worker.py $n 8 20 > gpurun_out/mp_P2_n$n.log 2>&1
  echo "mp P=2 n=$n rc=$?"; grep -E "MP OK|Error|error" gpurun_out/mp_P2_n$n.log | head -3
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29802 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scale_P2.json 2> gpurun_out/scale_P2.err; echo "bench P=2 rc=$?"
tail -1 gpurun_out/scale_P2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], '%.3e'%d['value']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items()]" 2>&1 | head -16
