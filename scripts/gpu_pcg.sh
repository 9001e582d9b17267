# PCG GPU tests + 512^3 PCG bench (stage table) + launch window traffic.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pcg.py -x -q -rs > gpurun_out/pytest_pcg.log 2>&1; echo "pcg rc=$?"; tail -4 gpurun_out/pytest_pcg.log
timeout 900 python bench.py --solver pcg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_pcg.json 2> gpurun_out/bench_pcg.err; echo "bench pcg rc=$?"
tail -1 gpurun_out/bench_pcg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks']); [print(k, round(v['ms_per_step'],3), v['launches'], v['alg_GBps']) for k,v in d['stages'].items() if k.startswith('pcg')]"
CMD="python bench.py --solver pcg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 5000 -c 100 --csv --log-file gpurun_out/launches_pcg512_t.csv $CMD > gpurun_out/ncu_launch_pcg.log 2>&1; echo "ncu launches rc=$?"
