mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
export NCU_KERNEL=k_push_key_brick NCU_OUT=push_key_p${NG} NCU_SKIP=3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29850 --no-python scripts/rank0_ncu.sh --gpus $NG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p4_ncu.log 2>&1; echo "ncu P=$NG rc=$?"
tail -3 gpurun_out/p4_ncu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_push_key_brick -s 3 -c 1 -o gpurun_out/push_key_p1mr -f env PIC_FORCE_MR=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p1_ncu.log 2>&1; echo "ncu P=1 MR rc=$?"
