#!/bin/bash
# torchrun --no-python wrapper: rank 0 runs under ncu (one kernel, full set), the others plain.
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNEL}" -s ${NCU_SKIP:-3} -c 1 -o gpurun_out/${NCU_OUT} -f python bench.py "$@"
else
  exec python bench.py "$@"
fi
