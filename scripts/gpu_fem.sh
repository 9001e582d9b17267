mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fem.py -x -q -rs > gpurun_out/pytest_fem.log 2>&1; echo "fem rc=$?"; tail -15 gpurun_out/pytest_fem.log
timeout 1200 python bench.py --solver fem --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fem.json 2> gpurun_out/bench_fem.err; echo "bench fem rc=$?"
tail -1 gpurun_out/bench_fem.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('pcg'), d['roofline']); [print(k, round(v['ms_per_step'],3), v['launches'], v['alg_GBps']) for k,v in d['stages'].items()]"
tail -3 gpurun_out/bench_fem.err
