# ncu DRAM / L2 hit counts of reorder_deposit with and without the L2 bulk prefetch
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex.sum
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for v in "$@"; do
  PIC_NVCC_EXTRA="$v" python -c "from paper_2605_05469_b200 import build_lib; build_lib(True)" > gpurun_out/build.log 2>&1 || { echo build failed; continue; }
  tag=$(echo "$v" | tr -dc 'A-Za-z0-9_=' | tr '=' '_')
  timeout 900 ncu --metrics $M --clock-control none -k regex:"reorder_deposit" -s 3 -c 2 --csv --log-file gpurun_out/pf_$tag.csv $CMD > /dev/null 2>&1; echo "ncu [$v] rc=$?"
  python - gpurun_out/pf_$tag.csv <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[1:]: print('  ', r[ki], r[vi], r[ui])
PY
done
