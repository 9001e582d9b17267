# place by cursor atomics + RED counts in the push (PIC_PLACE_ATOMIC=1) vs returned ranks (0)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "not damping" > gpurun_out/pl_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pl_pytest.log
PIC_FORCE_MR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or bit_exact or deposit or init" > gpurun_out/pl_pytest_mr.log 2>&1; echo "pytest MR rc=$?"; tail -1 gpurun_out/pl_pytest_mr.log
for v in "" "-DPIC_PLACE_ATOMIC=0" ""; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/pl.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pl.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('push_key','scan','place','reorder_deposit')})"
done
