# pencils on 2 GPUs (2x1) and slabs regression on 2 GPUs; then the 1-GPU parity subset
mkdir -p gpurun_out
export PYTHONPATH=$PWD
nvidia-smi -L
timeout 1200 python -m pytest tests/test_gpu_multirank.py -x -q -rs -k "pencil or (slab and 2)" > gpurun_out/pen2_pytest.log 2>&1; echo "multirank rc=$?"; tail -3 gpurun_out/pen2_pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pen2_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/pen2_parity.log
