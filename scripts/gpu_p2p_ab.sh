# 2 GPUs: bench P=2 under transport variants (env strings), stage table each.
mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
i=0
for v in "PIC_P2P=1" "$@"; do
  i=$((i+1))
  env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29810+i)) bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err; echo "== [$v] rc=$?"
  tail -1 gpurun_out/ab_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step']>0.2]" 2>&1 | head -16
done
