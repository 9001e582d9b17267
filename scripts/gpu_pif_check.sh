# PIF with the repo's own fine-grid FFT: parity tests, smoke, PIF bench line and its launch list
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_gpu_pif.py -x -q > gpurun_out/pif_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pif_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pif_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/pif_smoke.log
timeout 900 python bench.py --solver pif --n 512 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pif_bench.json 2> gpurun_out/pif_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/pif_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:round(v['ms_per_step'],2) for k,v in d['stages'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pif_launches.csv python bench.py --solver pif --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/pif_ncu.log 2>&1; echo "ncu rc=$?"; grep -c k_c2c gpurun_out/pif_launches.csv; grep -ci "regular_fft\|cufft" gpurun_out/pif_launches.csv
