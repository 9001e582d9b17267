# Round-end evidence on one B200: tests, bench line, ncu launch list + traffic, ncu full set.
mkdir -p gpurun_out
R=${ROUND:-r01}
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.max.mem --format=csv > gpurun_out/gpu_$R.txt
lscpu > gpurun_out/lscpu_$R.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$R.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$R.log
timeout 1200 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_$R.json | cut -c1-400
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$R.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$R.json | cut -c1-300
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain512_$R.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/launches_512_$R.csv $CMD > gpurun_out/ncu_launch_$R.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"reorder_deposit|push_key_brick" -s 4 -c 2 -o gpurun_out/full512_$R -f $CMD > gpurun_out/ncu_full_$R.log 2>&1; echo "ncu full rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fft|place" -s 12 -c 6 -o gpurun_out/full512fft_$R -f $CMD > gpurun_out/ncu_fullfft_$R.log 2>&1; echo "ncu full fft rc=$?"
