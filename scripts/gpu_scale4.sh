# Multi-GPU evidence on one box (run with gpurun --gpus 4): multirank tests, then the
# 512^3 bench at P = 1, 2, 4 for the FFT and the PCG solver.
mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l); echo "GPUs: $NG"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/pytest_mr4.log 2>&1; echo "mr rc=$?"; tail -4 gpurun_out/pytest_mr4.log
for S in fft pcg; do
for P in 1 2 4; do
  [ $P -le $NG ] || continue
  if [ $P -eq 1 ]; then CMD="python bench.py --solver $S --steps 5 --warmup 3 --no-cpu-baseline --no-e2e";
  else CMD="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $((29800+P)) bench.py --gpus $P --solver $S --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"; fi
  timeout 900 $CMD > gpurun_out/scale_${S}_P$P.json 2> gpurun_out/scale_${S}_P$P.err; echo "bench $S P=$P rc=$?"
  tail -1 gpurun_out/scale_${S}_P$P.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],2), '%.3e'%d['value'], d.get('nvlink')); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step'] > 0.05]" 2>&1 | head -20
done
done
