# pencils with the 24-B field pack: 4-GPU pencil parity + bench (and the slab bench for reference)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_gpu_multirank.py -q -rs -x -k "pencil" > gpurun_out/p4b_pytest.log 2>&1; echo "pencil pytest rc=$?"; tail -2 gpurun_out/p4b_pytest.log
timeout 900 python bench.py --gpus 4 --pgrid 2x2 --no-cpu-baseline > gpurun_out/p4b_bench_pencil.json 2> gpurun_out/p4b_bench_pencil.err; echo "bench pencil rc=$?"
timeout 900 python bench.py --gpus 4 --no-cpu-baseline > gpurun_out/p4b_bench_slab.json 2> gpurun_out/p4b_bench_slab.err; echo "bench slab rc=$?"
for f in pencil slab; do python -c "
import json; d=json.loads(open('gpurun_out/p4b_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],2), d['e2e']['value'] if d.get('e2e') else None, {k:round(v['ms_per_step'],2) for k,v in d['stages'].items() if v['ms_per_step']>0.05})"; done
