# A/B of NCCL environment settings on the 4-GPU 512^3 slab bench: step time and rank 0's xpose / exchange
mkdir -p gpurun_out
run() {
  echo "== [$*]"
  env "$@" timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nab.json 2> gpurun_out/nab.err || { echo fail; tail -3 gpurun_out/nab.err; return; }
  python -c "
import json; d=json.loads(open('gpurun_out/nab.json').read().strip().splitlines()[-1]); s=d['stages']
print(round(d['ms_per_step'],3), 'xpose', round(s['xpose']['ms_per_step'],3), 'exchange', round(s['exchange']['ms_per_step'],3))"
}
run X=0
run NCCL_MIN_NCHANNELS=16
run NCCL_MIN_NCHANNELS=32
run NCCL_NCHANNELS_PER_NET_PEER=8 NCCL_MIN_P2P_NCHANNELS=16
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=64
run NCCL_P2P_NVL_CHUNKSIZE=1048576
run NCCL_P2P_NVL_CHUNKSIZE=2097152 NCCL_MIN_P2P_NCHANNELS=16
run X=0
