# Round-end confirmation at HEAD: GPU suite, smoke, the default bench line and the reference arm.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/head_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/head_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/head_smoke.log
timeout 900 python bench.py > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/head_bench.json | cut -c1-250
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/head_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/head_ref.json | cut -c1-200
