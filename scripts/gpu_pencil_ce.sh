# 4 GPUs: pencils with copy-engine redistributions and transposes -- multi-rank parity, bench A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -rs > gpurun_out/pce_pytest.log 2>&1; echo "multirank rc=$?"; tail -2 gpurun_out/pce_pytest.log
for v in "PIC_PENCIL_PULL=1" "PIC_PENCIL_PULL=0" "PIC_PENCIL_PULL=0 PIC_XPOSE_PULL=0"; do
  env $v timeout 600 python bench.py --gpus 4 --pgrid 2x2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pce.json 2> gpurun_out/pce_$(echo $v | tr -dc 'A-Z0-9_=' | tr '=' '_').err || { echo fail; tail -3 gpurun_out/pce*.err; continue; }
  python -c "
import json; d=json.loads(open('gpurun_out/pce.json').read().strip().splitlines()[-1]); s=d['stages']
print('$v', round(d['ms_per_step'],3), 'xpose', round(s['xpose']['ms_per_step'],3), 'exchange', round(s['exchange']['ms_per_step'],3))"
done
