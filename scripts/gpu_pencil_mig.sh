# 4 GPUs: pencils with peer migration -- multi-rank parity, bench A/B
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -rs > gpurun_out/pmig_pytest.log 2>&1; echo "multirank rc=$?"; tail -2 gpurun_out/pmig_pytest.log
for v in "PIC_PENCIL_MIG=1" "PIC_PENCIL_MIG=0" "PIC_PENCIL_MIG=1"; do
  env $v timeout 600 python bench.py --gpus 4 --pgrid 2x2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pmig.json 2> gpurun_out/pmig.err || { echo fail; tail -3 gpurun_out/pmig.err; continue; }
  python -c "
import json; d=json.loads(open('gpurun_out/pmig.json').read().strip().splitlines()[-1]); s=d['stages']
print('$v', round(d['ms_per_step'],3), 'xpose', round(s['xpose']['ms_per_step'],3), 'exchange', round(s['exchange']['ms_per_step'],3), 'migrated/step', d['config']['migrated_per_step'])"
done
grep -h "stages ms/step" gpurun_out/pmig.err | sed "s/\[rank/\n[rank/g" | grep rank > gpurun_out/pmig_rank_stages.txt
