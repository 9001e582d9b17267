mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l); echo "GPUs: $NG"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs -x > gpurun_out/pytest_mig.log 2>&1; echo "mr rc=$?"; tail -3 gpurun_out/pytest_mig.log
for MIG in 0 1; do
  if [ $MIG = 1 ]; then export PIC_P2P_MIG=1; else unset PIC_P2P_MIG; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29830+MIG)) bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mig.json 2> gpurun_out/bench_mig.err; echo "bench MIG=$MIG rc=$?"
  tail -1 gpurun_out/bench_mig.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], '%.3e'%d['value']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step'] > 0.2]"
done
