# 1 GPU at HEAD: the -m gpu suite, smoke, the default bench line and the reference arm
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/c1_pytest.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/c1_smoke.log
timeout 1200 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/c1_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/c1_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/c1_ref.json | cut -c1-200
