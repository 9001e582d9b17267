# quick check: particle parity (P = 1 and the multi-rank instantiations forced), the bench line
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boris.py -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/q_pytest.log
PIC_FORCE_MR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or bit_exact or deposit or init" > gpurun_out/q_pytest_mr.log 2>&1; echo "pytest MR rc=$?"; tail -1 gpurun_out/q_pytest_mr.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/q_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
