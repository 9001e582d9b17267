mkdir -p gpurun_out
R=${ROUND:-r01}
CMD="python bench.py --solver pcg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 5000 -c 300 --csv --log-file gpurun_out/launches_pcg512_$R.csv $CMD > gpurun_out/ncu_launch_pcg.log 2>&1; echo "ncu launches rc=$?"
