# 4 GPUs: the whole multi-rank suite (slabs both transports, PCG/FEM, pencils 2x1 and 2x2; with the
# injected-charge solve vs the oracle) and the 4-GPU bench lines (slabs, pencils 2x2)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_gpu_multirank.py -q -rs -v > gpurun_out/mrf_pytest.log 2>&1; echo "multirank rc=$?"; tail -3 gpurun_out/mrf_pytest.log
timeout 900 python bench.py --gpus 4 > gpurun_out/mrf_bench_slab.json 2> gpurun_out/mrf_bench_slab.err; echo "bench slab rc=$?"
timeout 900 python bench.py --gpus 4 --pgrid 2x2 --no-cpu-baseline > gpurun_out/mrf_bench_pencil.json 2> gpurun_out/mrf_bench_pencil.err; echo "bench pencil rc=$?"
timeout 900 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/mrf_bench_slab2.json 2> gpurun_out/mrf_bench_slab2.err; echo "bench slab2 rc=$?"
for f in slab pencil slab2; do python -c "
import json; d=json.loads(open('gpurun_out/mrf_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],2), d['value'], d['e2e']['value'] if d.get('e2e') else None)"; done
