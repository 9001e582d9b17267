mkdir -p gpurun_out
timeout 900 python bench.py --solver pcg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_pcg.json 2> gpurun_out/bench_pcg.err; echo "bench pcg rc=$?"
tail -1 gpurun_out/bench_pcg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['pcg'], d['roofline']); [print(k, round(v['ms_per_step'],3), v['launches'], v['alg_GBps']) for k,v in d['stages'].items()]"
tail -3 gpurun_out/bench_pcg.err
