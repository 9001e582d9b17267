mkdir -p gpurun_out
(nproc; free -g; lscpu | head -30; nvidia-smi; cat /proc/meminfo | head -3) > gpurun_out/host_probe.txt 2>&1
export PYTHONPATH=$PWD
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_base_bench.json 2> gpurun_out/r02_base_bench.err; echo "bench rc=$?"
