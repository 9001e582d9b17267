# Round 2: full GPU suite (incl. 256^3 element-wise solve parity and the 1024^3 x 1 run), smoke,
# the default bench line (cpu_baseline with both oracle legs) and the reference arm.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python -c "from paper_2605_05469_b200._build import build_lib; build_lib()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu -rs --durations=15 > gpurun_out/r02_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02_bench.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02_ref.json | cut -c1-300
