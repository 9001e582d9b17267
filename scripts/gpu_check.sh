mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g | head -2; nproc; lscpu | grep -E "Model name|Socket|Core|Thread" 
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --n 128 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench128.log 2>&1; echo "bench128 rc=$?"; tail -3 gpurun_out/bench128.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench512.log 2>&1; echo "bench512 rc=$?"; tail -5 gpurun_out/bench512.log
