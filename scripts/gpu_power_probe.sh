# Clocks/power of all GPUs while the P=1 and P=4 benches run (diagnostics).
mkdir -p gpurun_out
NG=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
probe() { nvidia-smi --query-gpu=index,clocks.sm,clocks.mem,power.draw,power.limit,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/power_$1.csv & echo $!; }
P1=$(probe p1); timeout 600 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pp1.json 2>/dev/null; kill $P1
PN=$(probe pn); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29901 bench.py --gpus $NG --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ppn.json 2> gpurun_out/ppn.err; kill $PN
for f in pp1 ppn; do tail -1 gpurun_out/$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['stages'].items() if v['ms_per_step']>1})"; done
python - <<'PY'
import csv, statistics
for tag in ("p1", "pn"):
    rows = [r for r in csv.reader(open(f"gpurun_out/power_{tag}.csv")) if len(r) >= 6]
    by = {}
    for r in rows:
        try:
            by.setdefault(r[0].strip(), []).append((float(r[1].split()[0]), float(r[2].split()[0]), float(r[3].split()[0]), r[5].strip()))
        except Exception:
            pass
    for g, v in sorted(by.items()):
        busy = [x for x in v if x[2] > 300]
        if not busy: continue
        print(tag, "gpu", g, "n", len(busy), "sm", statistics.median(x[0] for x in busy), "mem", statistics.median(x[1] for x in busy),
              "W med", statistics.median(x[2] for x in busy), "W max", max(x[2] for x in busy), "reasons", sorted(set(x[3] for x in busy))[:3])
PY
