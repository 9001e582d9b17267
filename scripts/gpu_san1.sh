# compute-sanitizer (memcheck, racecheck, synccheck) on a 16^3 run + PIF (1 GPU); flush-cost probe
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_${tool}_p1.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE RUN OK" gpurun_out/san_${tool}_p1.log | head -3
done
for v in "" "-DPIC_RD_SKIP_FLUSH"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/fl.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/fl.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['stages'].items() if k in ('push_key','place','reorder_deposit')})"
done
python -c "from paper_2605_05469_b200._build import build_lib; build_lib(force=True)" > /dev/null 2>&1
