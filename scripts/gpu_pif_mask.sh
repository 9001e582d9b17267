# PIF: own bin scan (no cub) and plane-masked fine-grid x / y passes -- 1-GPU PIF suite, decomposed
# PIF parity on 2 and 4 GPUs, PIF bench on 1, 2, 4 GPUs
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_pif.py -q -x > gpurun_out/pm_pif1.log 2>&1; echo "pif 1-GPU rc=$?"; tail -1 gpurun_out/pm_pif1.log
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -rs -k "pif" > gpurun_out/pm_pytest.log 2>&1; echo "pif multirank rc=$?"; tail -1 gpurun_out/pm_pytest.log
for g in 1 2 4; do
  timeout 1200 python bench.py --solver pif --gpus $g --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/pm_bench_$g.json 2> gpurun_out/pm_bench_$g.err; echo "bench pif $g rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/pm_bench_$g.json').read().strip().splitlines()[-1]); print($g, d['n_gpus'], round(d['ms_per_step'],1), d['value'], {k:round(v['ms_per_step'],1) for k,v in d['stages'].items()})"
done
