# BJ config 5 (FD-PCG) and the FEM solver at HEAD: 512^3 x 8 on 1 and 4 GPUs
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for solver in pcg fem; do
  for g in 1 4; do
    timeout 1500 python bench.py --solver $solver --gpus $g --steps 3 --warmup 3 --no-e2e $( [ $g -gt 1 ] && echo --no-cpu-baseline ) > gpurun_out/cg_${solver}_$g.json 2> gpurun_out/cg_${solver}_$g.err; echo "$solver $g rc=$?"
    python -c "
import json; d=json.loads(open('gpurun_out/cg_${solver}_$g.json').read().strip().splitlines()[-1]); print('$solver', d['n_gpus'], round(d['ms_per_step'],1), d['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d.get('pcg'))"
  done
done
