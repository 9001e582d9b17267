mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs -k "cg_solvers" > gpurun_out/pytest_mrcg.log 2>&1; echo "mr cg rc=$?"; tail -4 gpurun_out/pytest_mrcg.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29815 bench.py --gpus 2 --solver fem --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench2_fem.json 2> gpurun_out/bench2_fem.err; echo "bench2 fem rc=$?"
tail -1 gpurun_out/bench2_fem.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], '%.3e'%d['value'], d.get('pcg'))"
