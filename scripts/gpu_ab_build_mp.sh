# A/B of compile-time variants on the P-rank 512^3 bench (all GPUs of the box).
mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
i=0
for v in "" "$@"; do
  i=$((i+1))
  echo "== variant [$v]"
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200 import build_lib; build_lib(True)" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; continue; }
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29830+i)) bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abm_$i.json 2> gpurun_out/abm_$i.err
  tail -1 gpurun_out/abm_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step']>0.3]" 2>&1 | head -16
done
