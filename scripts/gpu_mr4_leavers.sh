# larger leaver staging + warp-aggregated overflow: multi-rank parity (4 GPUs) and 4-GPU benches
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_gpu_multirank.py -q -rs -x > gpurun_out/lv_pytest.log 2>&1; echo "multirank rc=$?"; tail -2 gpurun_out/lv_pytest.log
timeout 900 python bench.py --gpus 4 --no-cpu-baseline --no-e2e > gpurun_out/lv_bench_slab.json 2> gpurun_out/lv_bench_slab.err; echo "bench slab rc=$?"
timeout 900 python bench.py --gpus 4 --pgrid 2x2 --no-cpu-baseline --no-e2e > gpurun_out/lv_bench_pencil.json 2> gpurun_out/lv_bench_pencil.err; echo "bench pencil rc=$?"
timeout 900 python bench.py --gpus 2 --no-cpu-baseline --no-e2e > gpurun_out/lv_bench_slab2.json 2> gpurun_out/lv_bench_slab2.err; echo "bench slab2 rc=$?"
for f in slab pencil slab2; do python -c "
import json; d=json.loads(open('gpurun_out/lv_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['stages'].items() if v['ms_per_step']>0.05})"; done
grep -c "NCCL INFO" gpurun_out/lv_bench_slab.err; grep "NCCL INFO" gpurun_out/lv_bench_slab.err | grep -m2 -i "nranks"
