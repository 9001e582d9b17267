# Evidence for BJ config 5 (PCG) at 512^3 on one B200: bench line (with cpu_baseline, e2e),
# ncu launch window (time + DRAM bytes), ncu --set full of one SSOR half-sweep and one matvec.
mkdir -p gpurun_out
timeout 1500 python bench.py --solver pcg --steps 5 --warmup 3 > gpurun_out/bench_pcg_r01.json 2> gpurun_out/bench_pcg_r01.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_pcg_r01.json | cut -c1-300
CMD="python bench.py --solver pcg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 9000 -c 400 --csv --log-file gpurun_out/launches_pcg512_r01.csv $CMD > gpurun_out/ncu_launch_pcg.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sor|k_pcg_matvec|k_pcg_update" -s 3000 -c 4 -o gpurun_out/full_pcg512_r01 -f $CMD > gpurun_out/ncu_full_pcg.log 2>&1; echo "ncu full rc=$?"
