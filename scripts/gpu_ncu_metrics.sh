# Selected ncu metrics of one kernel launch at 512^3 (after the same command ran clean).
mkdir -p gpurun_out
CMD="python bench.py --n ${N:-512} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_m.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics ${NCU_M:-gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active} --clock-control none -k regex:"${NCU_K:-reorder}" -s ${NCU_S:-3} -c ${NCU_C:-1} --csv $CMD > gpurun_out/ncu_m.csv 2> gpurun_out/ncu_m.err; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/ncu_m.csv')) if len(r) > 10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d['Kernel Name'][:40], d['Metric Name'], d['Metric Unit'], d['Metric Value'])
PY
