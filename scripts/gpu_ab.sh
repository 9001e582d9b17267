mkdir -p gpurun_out
for v in 3 4 5; do
PIC_REORDER_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or push_bit or sort_keys" > gpurun_out/pytest_v$v.log 2>&1; echo "pytest v$v rc=$?"
PIC_REORDER_VARIANT=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench512_v$v.log 2>&1; echo "variant $v rc=$?"; tail -1 gpurun_out/bench512_v$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value']); [print(k, round(v['ms_per_step'],3), v['alg_GBps']) for k,v in d['stages'].items() if k in ('reorder_deposit',)]"
done
