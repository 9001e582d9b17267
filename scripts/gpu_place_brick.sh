# place per source brick (offs of the 27 neighbouring bricks in shared memory): parity + A/B + ncu L2 requests
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boris.py tests/test_gpu_pcg.py -x -q > gpurun_out/pb_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pb_pytest.log
PIC_FORCE_MR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twenty or bit_exact or deposit or init" > gpurun_out/pb_pytest_mr.log 2>&1; echo "pytest MR rc=$?"; tail -1 gpurun_out/pb_pytest_mr.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "512" > gpurun_out/pb_full.log 2>&1; echo "fullsize rc=$?"; tail -1 gpurun_out/pb_full.log
for v in 1 0 1; do
  PIC_PLACE_BRICK=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/pb.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pb.json').read().strip().splitlines()[-1]); print('brick=$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('push_key','scan','place','reorder_deposit')})"
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum --clock-control none -k regex:place -c 8 --csv --log-file gpurun_out/place_launches.csv $CMD > gpurun_out/place_ncu.log 2>&1; echo "ncu rc=$?"
