# ncu --set full of selected kernels at 512^3 (after the same command ran clean).
mkdir -p gpurun_out
CMD="python bench.py --n 512 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain512.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-fft}" -s ${NCU_S:-0} -c ${NCU_C:-5} -o gpurun_out/${NCU_O:-prof512} -f $CMD > gpurun_out/ncu512.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu512.log
