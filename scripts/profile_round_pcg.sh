# Round-end evidence for BJ config 5 (PCG) on one B200: bench line, ncu launch window, ncu full set.
mkdir -p gpurun_out
R=${ROUND:-r01}
timeout 1500 python bench.py --solver pcg --steps 5 --warmup 3 > gpurun_out/bench_pcg_$R.json 2> gpurun_out/bench_pcg_$R.err; echo "bench pcg rc=$?"; tail -1 gpurun_out/bench_pcg_$R.json | cut -c1-300
CMD="python bench.py --solver pcg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 9000 -c 300 --csv --log-file gpurun_out/launches_pcg512_$R.csv $CMD > gpurun_out/ncu_launch_pcg.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sor4|k_pcg_matvec8|k_pcg_update4|k_pcg_gradient8|k_pcg_resid0_8" -s 40 -c 5 -o gpurun_out/full_pcg512_$R -f $CMD > gpurun_out/ncu_full_pcg.log 2>&1; echo "ncu full rc=$?"
