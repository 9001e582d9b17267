# 2-GPU: multirank tests (FFT both transports + PCG) and the 512^3 bench for both solvers.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/pytest_mr.log 2>&1; echo "mr rc=$?"; tail -5 gpurun_out/pytest_mr.log
for S in fft pcg; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 --solver $S --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench2_$S.json 2> gpurun_out/bench2_$S.err; echo "bench2 $S rc=$?"
  tail -1 gpurun_out/bench2_$S.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], '%.3e'%d['value'], d.get('pcg')); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items()]"
done
