mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench512.log 2>&1; echo "bench512 rc=$?"; tail -1 gpurun_out/bench512.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value']); [print(k, round(v['ms_per_step'],3), v['alg_GBps']) for k,v in d['stages'].items()]"
CMD="python bench.py --n 256 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain256.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-fft}" -s ${NCU_S:-8} -c ${NCU_C:-5} -o gpurun_out/prof256c -f $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu.log
