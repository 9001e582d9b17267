# A/B of one environment switch on the 512^3 bench stage table: bash gpu_ab_env.sh VAR=val
mkdir -p gpurun_out
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); [print(' ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items()]"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_quick.log
for v in "" "$@"; do
  echo "== variant [$v]"
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1 && show gpurun_out/ab.log
done
