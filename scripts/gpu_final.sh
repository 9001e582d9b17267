# The driver's round-end commands on one B200 (tests, smoke, bench, reference arm) plus the
# PIF bench line and its ncu evidence.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_ref.json | cut -c1-200
timeout 900 python bench.py --solver pif --steps 3 --warmup 3 > gpurun_out/final_bench_pif.json 2> gpurun_out/final_bench_pif.err; echo "bench pif rc=$?"; tail -1 gpurun_out/final_bench_pif.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_pif512_binned.csv python bench.py --solver pif --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pif_launch2.log 2>&1; echo "ncu launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_interp_tiled -c 1 -o gpurun_out/full_pif512_interp python scripts/pif_time.py 512 8 > gpurun_out/ncu_pif512_interp.log 2>&1; echo "ncu interp rc=$?"
