# FFT transposes by peer pulls (PIC_XPOSE_PULL=1) vs ncclAlltoAll: slab parity at 2 and 4 GPUs, 4-GPU A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
PIC_XPOSE_PULL=1 timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -rs -x -k "slab_decomposition_matches and peer" > gpurun_out/xp_pytest.log 2>&1; echo "pull parity rc=$?"; tail -1 gpurun_out/xp_pytest.log
for v in 1 0 1 0; do
  PIC_XPOSE_PULL=$v timeout 900 python bench.py --gpus 4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/xp_$v.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/xp_$v.json').read().strip().splitlines()[-1]); print('pull=$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('xpose','exchange','fft_z_mul')}, round(d['nvlink']['xpose_GBps'],1))"
done
