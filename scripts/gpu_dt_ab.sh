mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
for DT in 0.05 0.0001; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29840 bench.py --gpus $NG --dt $DT --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_dt.json 2> gpurun_out/bench_dt.err; echo "bench dt=$DT rc=$?"
  tail -1 gpurun_out/bench_dt.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['migrated_per_step']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step'] > 0.2]"
  grep stages gpurun_out/bench_dt.err | cut -c1-250
done
