# Round-2 evidence on one B200 (profile_round.sh with ROUND=r02: GPU suite, smoke, bench line with
# cpu_baseline + e2e, reference arm, ncu launch list with DRAM bytes and L2 requests, ncu full sets),
# then the PIF bench line and the bench with the oracle leg on the 512^3 configuration itself.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
ROUND=r02 bash scripts/profile_round.sh
timeout 900 python bench.py --solver pif --steps 3 --warmup 3 > gpurun_out/bench_pif_r02.json 2> gpurun_out/bench_pif_r02.err; echo "bench pif rc=$?"; tail -1 gpurun_out/bench_pif_r02.json | cut -c1-300
timeout 1500 python bench.py --cpu-full --no-e2e > gpurun_out/bench_cpufull_r02.json 2> gpurun_out/bench_cpufull_r02.err; echo "bench cpu-full rc=$?"; tail -1 gpurun_out/bench_cpufull_r02.json | cut -c1-300
