# Evidence for the coalesced place mapping: full GPU suite, smoke, the 512^3 FFT bench line,
# and its ncu launch list (with DRAM bytes) at 1 timed step.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/place_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/place_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/place_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/place_smoke.log
timeout 900 python bench.py > gpurun_out/place_bench.json 2> gpurun_out/place_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/place_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks']); [print(k, round(v['ms_per_step'],3), v['alg_GBps']) for k,v in d['stages'].items()]"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum --clock-control none --csv --log-file gpurun_out/place_launches512.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/place_ncu.log 2>&1; echo "ncu rc=$?"
