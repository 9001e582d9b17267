# A/B of compile-time variants on the 512^3 bench: bash gpu_ab_build.sh "-DA=1" "-DA=2 -DB=3" ...
mkdir -p gpurun_out
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); [print(' ', k, round(v['ms_per_step'],3)) for k,v in d['stages'].items() if v['ms_per_step'] > 0.3]"; }
for v in "" "$@"; do
  echo "== variant [$v]"
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200 import build_lib; build_lib(True)" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; continue; }
  if [ -n "$AB_TEST" ]; then timeout 900 python -m pytest $AB_TEST -m gpu -x -q 2>&1 | tail -1; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ab.log 2>&1 && show gpurun_out/ab.log
done
