# reorder_deposit A/B: chunk capacity / CTAs per SM of the pipelined kernel (bench stage times)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in "-DPIC_RD_CAP=640 -DPIC_RD_MINB=3" "-DPIC_RD_CAP=896 -DPIC_RD_MINB=2" "-DPIC_RD_CAP=1024 -DPIC_RD_MINB=2" "-DPIC_RD_CAP=448 -DPIC_RD_MINB=4"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/rdab.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/rdab.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['stages'].items() if k in ('push_key','place','reorder_deposit')})"
done
