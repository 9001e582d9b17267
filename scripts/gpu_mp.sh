mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_mp.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_mp.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench512_p1.log 2>&1; echo "bench p1 rc=$?"; tail -1 gpurun_out/bench512_p1.log | cut -c1-200
