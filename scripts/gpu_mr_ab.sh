mkdir -p gpurun_out
for MR in 0 1; do
  if [ $MR = 1 ]; then export PIC_FORCE_MR=1; else unset PIC_FORCE_MR; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_mr.log 2>&1
  echo "== FORCE_MR=$MR"; tail -1 gpurun_out/ab_mr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); [print(' ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step'] > 0.3]"
done
