# 1024^3 grid on 4 GPUs: 4 ppc (4.3e9 particles), pencils 2x2 and slabs 1x4, 300 steps with the damping fit
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for pg in 2x2 1x4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29911 scripts/mp_damping.py 1024 4 300 15 $pg > gpurun_out/d1024_$pg.log 2>&1; echo "$pg rc=$?"; grep '^{' gpurun_out/d1024_$pg.log | cut -c1-400
done
