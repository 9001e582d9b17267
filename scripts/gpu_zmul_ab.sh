# z pass: the two inverse transforms fused into one 2TW-line call (PIC_ZMUL_FUSED) -- solve parity + A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in "" "-DPIC_ZMUL_FUSED=1 -DPIC_ZMUL_DIRECT=1" "-DPIC_ZMUL_FUSED=1"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "solve or twenty" > gpurun_out/zm_pytest.log 2>&1; echo "[$v] pytest rc=$?"; tail -1 gpurun_out/zm_pytest.log
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/zm.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/zm.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k.startswith('fft')})"
done
python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
