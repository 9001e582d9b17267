# Dev loop on a 2-GPU box: 1-GPU parity tests + 512^3 bench, then 2-rank parity (both transports) + P=2 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1; echo "bench P=1 rc=$?"
tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); [print('   ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step']>0.05]"
bash scripts/gpu_mp2ab.sh 2>&1 | grep -v "Warning\|return func"
