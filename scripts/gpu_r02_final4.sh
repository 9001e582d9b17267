# Round-2 4-GPU evidence at HEAD: multi-rank suite, benches (slabs, pencils 2x2, 2 GPUs), per-rank
# stage tables, and the 1024^3 x 4 ppc damping runs (pencils 2x2, slabs 1x4)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
bash scripts/gpu_mr4_final.sh
for f in slab pencil slab2; do grep -h "stages ms/step" gpurun_out/mrf_bench_$f.err | sed "s/\[rank/\n[rank/g" | grep rank; done > gpurun_out/mrf_rank_stages.txt
bash scripts/gpu_1024_4gpu.sh
