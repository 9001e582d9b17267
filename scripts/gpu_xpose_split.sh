# 4 GPUs: transposes overlapped with the y / z pass halves (PIC_XPOSE_SPLIT) -- parity, bench A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -rs > gpurun_out/split_pytest.log 2>&1; echo "multirank rc=$?"; tail -2 gpurun_out/split_pytest.log
for v in "PIC_XPOSE_SPLIT=1" "PIC_XPOSE_SPLIT=0" "PIC_XPOSE_SPLIT=1" "PIC_XPOSE_SPLIT=0"; do
 for pg in 1x4 2x2; do
  env $v timeout 600 python bench.py --gpus 4 --pgrid $pg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/split.json 2> gpurun_out/split.err || { echo fail; tail -3 gpurun_out/split.err; continue; }
  python -c "
import json; d=json.loads(open('gpurun_out/split.json').read().strip().splitlines()[-1]); s=d['stages']
print('$v $pg', round(d['ms_per_step'],3), 'xpose', round(s['xpose']['ms_per_step'],3), 'y_fwd', round(s['fft_y_fwd']['ms_per_step'],3), 'z_mul', round(s['fft_z_mul']['ms_per_step'],3), 'launches', d['gpu_launches'])"
 done
done
