# Round-end evidence for the CG solvers on one B200: full GPU test suite, bench lines
# (PCG = BJ config 5, FEM = NEXT-4), ncu launch windows and full sets.
mkdir -p gpurun_out
R=${ROUND:-r01}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$R.log
timeout 1500 python bench.py --solver pcg --steps 5 --warmup 3 > gpurun_out/bench_pcg_$R.json 2> gpurun_out/bench_pcg_$R.err; echo "bench pcg rc=$?"; tail -1 gpurun_out/bench_pcg_$R.json | cut -c1-200
timeout 1500 python bench.py --solver fem --steps 3 --warmup 3 --cpu-steps 5 > gpurun_out/bench_fem_$R.json 2> gpurun_out/bench_fem_$R.err; echo "bench fem rc=$?"; tail -1 gpurun_out/bench_fem_$R.json | cut -c1-200
CMD="python bench.py --solver pcg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 5000 -c 300 --csv --log-file gpurun_out/launches_pcg512_$R.csv $CMD > gpurun_out/ncu_launch_pcg.log 2>&1; echo "ncu launches pcg rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sor4|k_pcg_matvec8|k_pcg_update4|k_pcg_gradient8|k_pcg_resid0_8" -s 40 -c 5 -o gpurun_out/full_pcg512_$R -f $CMD > gpurun_out/ncu_full_pcg.log 2>&1; echo "ncu full pcg rc=$?"
CMD="python bench.py --solver fem --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fem_matvec|k_fem_update" -s 20 -c 2 -o gpurun_out/full_fem512_$R -f $CMD > gpurun_out/ncu_full_fem.log 2>&1; echo "ncu full fem rc=$?"
