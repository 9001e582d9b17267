mkdir -p gpurun_out
CMD="python bench.py --n 256 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain256.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft|place" -s 8 -c 6 -o gpurun_out/prof_fft256 -f $CMD > gpurun_out/ncu_fft.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_fft.log
