# 4 GPUs: the whole multi-rank suite (slabs both transports, PCG/FEM, pencils 2x2) and
# 512^3 benches: slab 1x4 vs pencil 2x2, through bench.py --gpus 4 (self-launch under torchrun)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
nvidia-smi -L
timeout 1800 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/mr4_pytest.log 2>&1; echo "multirank rc=$?"; tail -3 gpurun_out/mr4_pytest.log
timeout 900 python bench.py --gpus 4 --no-cpu-baseline > gpurun_out/mr4_bench_slab.json 2> gpurun_out/mr4_bench_slab.err; echo "bench slab rc=$?"; tail -1 gpurun_out/mr4_bench_slab.json | cut -c1-400
grep -m3 "NCCL INFO.*nranks\|comm .* nRanks\|Init COMPLETE" gpurun_out/mr4_bench_slab.err
timeout 900 python bench.py --gpus 4 --pgrid 2x2 --no-cpu-baseline > gpurun_out/mr4_bench_pencil.json 2> gpurun_out/mr4_bench_pencil.err; echo "bench pencil rc=$?"; tail -1 gpurun_out/mr4_bench_pencil.json | cut -c1-400
