mkdir -p gpurun_out
python scripts/pcg_prof.py 256 > gpurun_out/pcgprof.log 2>&1; echo rc=$?; cat gpurun_out/pcgprof.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ssor_tb" -s 1 -c 1 -o gpurun_out/ssor_tb -f python scripts/pcg_prof.py 256 > gpurun_out/ncu_tb.log 2>&1; echo "ncu tb rc=$?"
PIC_PCG_TB=0 timeout 600 ncu --set full --clock-control none -k regex:"k_sor" -s 4 -c 1 -o gpurun_out/ssor_hs -f python scripts/pcg_prof.py 256 > gpurun_out/ncu_hs.log 2>&1; echo "ncu hs rc=$?"
