# FFT z pass A/B (input buffer vs direct stage-0 loads) and an ncu full capture of the solve passes
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in "" "-DPIC_ZMUL_DIRECT=1" "-DPIC_ZMUL_DIRECT=1 -DPIC_ZMUL_MINB=3"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/fab.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/fab.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k.startswith('fft') or k=='reorder_deposit'})"
done
python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fft_z_mul|k_fft_x_inv|k_fft_y|k_fft_x_fwd" -c 5 -o gpurun_out/r02_full_fft512 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fft.log 2>&1; echo "ncu rc=$?"
