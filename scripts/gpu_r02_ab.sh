# quick check: parity (also with the multi-rank kernel instantiations forced at P = 1), the bench line
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab_pytest.log
PIC_FORCE_MR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or bit_exact or deposit" > gpurun_out/ab_pytest_mr.log 2>&1; echo "pytest MR rc=$?"; tail -1 gpurun_out/ab_pytest_mr.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/ab_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
