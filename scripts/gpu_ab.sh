mkdir -p gpurun_out
for kb in 2 4 8; do
PIC_REORDER_KB=$kb timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench512_kb$kb.log 2>&1; echo "kb $kb rc=$?"; tail -1 gpurun_out/bench512_kb$kb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value']); [print(k, round(v['ms_per_step'],3), v['alg_GBps']) for k,v in d['stages'].items() if k in ('reorder_deposit',)]"
done
