# y passes compiled for 3 resident CTAs (80 registers, small spills) vs 2 -- solve parity + A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in "" "-DPIC_FFTY_MINB=3"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "solve" > gpurun_out/fy_pytest.log 2>&1; echo "[$v] pytest rc=$?"; tail -1 gpurun_out/fy_pytest.log
  for r in 1 2; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/fy.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/fy.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k.startswith('fft')})"
  done
done
python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
