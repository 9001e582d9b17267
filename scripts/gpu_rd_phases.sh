# reorder_deposit phase costs: rebuild with diagnostic knobs, bench stage times (parity is NOT kept)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in "" "-DPIC_RD_SKIP_RANK" "-DPIC_RD_SKIP_DEPOSIT" "-DPIC_RD_SKIP_RANK -DPIC_RD_SKIP_DEPOSIT" "-DPIC_RD_CAP=960 -DPIC_RD_MINB=4"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/ph.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ph.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['stages'].items() if k in ('push_key','place','reorder_deposit')})"
done
