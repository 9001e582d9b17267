# UBLKRED row flush of the deposit tile + x C2R pass direct loads: parity, MR-forced parity, A/B bench
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_fem.py -x -q > gpurun_out/bk_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/bk_pytest.log
PIC_FORCE_MR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or bit_exact or deposit or init" > gpurun_out/bk_pytest_mr.log 2>&1; echo "pytest MR rc=$?"; tail -1 gpurun_out/bk_pytest_mr.log
for v in "" "-DPIC_RD_BULK=0" "-DPIC_XINV_DIRECT=1"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bk.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bk.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('push_key','place','reorder_deposit','fft_x_inv')})"
done
python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
