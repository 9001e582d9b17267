# Round-2 evidence at HEAD on one B200: profile_round.sh (GPU suite, smoke, bench line, reference arm,
# ncu launch list + full sets) and the PIF bench line
mkdir -p gpurun_out
export PYTHONPATH=$PWD
ROUND=r02 bash scripts/profile_round.sh
timeout 900 python bench.py --solver pif --steps 3 --warmup 3 > gpurun_out/bench_pif_r02.json 2> gpurun_out/bench_pif_r02.err; echo "bench pif rc=$?"; tail -1 gpurun_out/bench_pif_r02.json | cut -c1-300
