# reorder_deposit: L2 prefetch of the next chunk's sources during the deposit (PIC_RD_PREFETCH) -- parity + A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pf_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pf_pytest.log
PIC_FORCE_MR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or bit_exact or deposit or init" > gpurun_out/pf_pytest_mr.log 2>&1; echo "pytest MR rc=$?"; tail -1 gpurun_out/pf_pytest_mr.log
for v in "" "-DPIC_RD_PREFETCH=0" "" "-DPIC_RD_PREFETCH=0"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/pf.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pf.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('push_key','place','reorder_deposit')})"
done
python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
