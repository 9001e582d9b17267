# 4-GPU check after the place change: multi-rank parity tests and the 4-GPU 512^3 bench.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/mp4_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/mp4_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/mp4_bench.json 2> gpurun_out/mp4_bench.err; echo "bench4 rc=$?"
tail -1 gpurun_out/mp4_bench.json | cut -c1-400
