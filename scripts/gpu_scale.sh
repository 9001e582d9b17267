# Multi-GPU checks + scaling on the GPUs of this box (run under gpurun --gpus N).
mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
echo "GPUs: $NG"
if [ "${RUN_PYTEST:-1}" = 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_scale.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_scale.log
fi
for P in 2 4 8; do
  [ $P -le $NG ] || continue
  for n in 32 64; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 --master-port $((29700+P+n)) tests/mp_worker.py $n 8 20 > gpurun_out/mp_P${P}_n$n.log 2>&1
    echo "mp P=$P n=$n rc=$?"; grep -E "MP OK|Error|error" gpurun_out/mp_P${P}_n$n.log | head -3
  done
done
for P in 1 2 4 8; do
  [ $P -le $NG ] || continue
  if [ $P -eq 1 ]; then CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e";
  else CMD="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $((29800+P)) bench.py --gpus $P --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"; fi
  timeout 900 $CMD > gpurun_out/scale_P$P.json 2> gpurun_out/scale_P$P.err; echo "bench P=$P rc=$?"
  tail -1 gpurun_out/scale_P$P.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], '%.3e'%d['value'], d['config'].get('migrated_per_step')); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items()]" 2>&1 | head -16
done
