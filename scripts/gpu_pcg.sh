# PCG GPU tests + FFT regression subset.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pcg.py -x -q -rs > gpurun_out/pytest_pcg.log 2>&1; echo "pcg rc=$?"; tail -15 gpurun_out/pytest_pcg.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_parity.log
