# PCG GPU tests + 512^3 PCG bench (stage table) + A/B of the 2- and 4-element SOR kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_boris.py -x -q -rs > gpurun_out/pytest_pcg.log 2>&1; echo "pcg+boris rc=$?"; tail -15 gpurun_out/pytest_pcg.log
for SOR2 in 0 1; do
PIC_PCG_SOR2=$SOR2 timeout 900 python bench.py --solver pcg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_pcg.json 2> gpurun_out/bench_pcg.err; echo "bench pcg SOR2=$SOR2 rc=$?"
tail -1 gpurun_out/bench_pcg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks']); [print(k, round(v['ms_per_step'],3), v['launches'], v['alg_GBps']) for k,v in d['stages'].items() if k.startswith('pcg')]"
done
