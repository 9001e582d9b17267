# 4 GPUs: transposes by copy-engine pulls (PIC_XPOSE_PULL=2) -- multi-rank parity, then bench A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
PIC_XPOSE_PULL=2 timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -x -k "not pif" > gpurun_out/ce_pytest.log 2>&1; echo "multirank CE rc=$?"; tail -2 gpurun_out/ce_pytest.log
for v in 0 2 1 2 0; do
  PIC_XPOSE_PULL=$v timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ce.json 2> gpurun_out/ce.err || { echo fail; tail -3 gpurun_out/ce.err; continue; }
  python -c "
import json; d=json.loads(open('gpurun_out/ce.json').read().strip().splitlines()[-1]); s=d['stages']
print('PULL=$v', round(d['ms_per_step'],3), 'xpose', round(s['xpose']['ms_per_step'],3), 'exchange', round(s['exchange']['ms_per_step'],3))"
done
