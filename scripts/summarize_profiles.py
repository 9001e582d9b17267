"""Turn the round's raw ncu outputs (gpurun_out/) into the committed summaries (profiles/)."""
import csv, io, json, os, re, subprocess, sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
G, P = "gpurun_out", "profiles"
os.makedirs(P, exist_ok=True)

# 1. launch list at the bench config (512^3 x 8): per-launch time and DRAM bytes
rows = [l for l in open(f"{G}/launches_512_{R}.csv") if l.startswith('"')]
rd = list(csv.DictReader(io.StringIO("".join(rows))))
launch = {}
for r in rd:
    k = int(r["ID"])
    kn = r["Kernel Name"]
    depth, cut = 0, len(kn)
    for i in range(len(kn) - 1, -1, -1):      # strip the trailing (parameter list)
        depth += kn[i] == ")"
        depth -= kn[i] == "("
        if depth == 0:
            cut = i
            break
    name = kn[:cut].replace("unnamed>::", "").replace("void ", "")
    d = launch.setdefault(k, {"id": k, "kernel": name, "grid": r["Grid Size"], "block": r["Block Size"]})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    if r["Metric Name"] == "gpu__time_duration.sum":
        d["time_us"] = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(unit, v)
    elif r["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r["Metric Name"].split(".")[0].replace("dram__bytes_", "dram_")] = v * scale
out = sorted(launch.values(), key=lambda d: d["id"])
with open(f"{P}/{R}_launches_512.csv", "w") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "time_us", "dram_read_bytes", "dram_write_bytes"])
    for d in out:
        w.writerow([d["id"], d["kernel"], d["grid"], d["block"], round(d.get("time_us", 0), 2),
                    int(d.get("dram_read", 0)), int(d.get("dram_write", 0))])
# per-kernel share of one step (cold-cache, serialised: compare shares)
agg = {}
for d in out:
    a = agg.setdefault(d["kernel"], [0, 0.0, 0.0])
    a[0] += 1; a[1] += d.get("time_us", 0); a[2] += d.get("dram_read", 0) + d.get("dram_write", 0)
tot = sum(a[1] for a in agg.values())
lines = [f"# {R}: ncu launch list, 512^3 x 8 ppc (bench config), gpu__time_duration + dram bytes, "
         f"--clock-control none; {len(out)} launches after skipping init", "kernel,launches,total_us,share,GB_per_launch,GBps"]
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{n},{t:.1f},{t / tot:.3f},{b / n / 1e9:.3f},{b / (t * 1e-6) / 1e9 if t else 0:.0f}")
open(f"{P}/{R}_launches_512_summary.csv", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
# traffic per launch of the dominant kernel for bench.py
tr = {k: (b / n) for k, (n, t, b) in agg.items()}
json.dump({"landau3d_512^3x8ppc_fft": {"reorder_deposit": tr.get("k_reorder_deposit", None),
                                        "push_key_brick": tr.get("k_push_key_brick", None),
                                        "source": f"profiles/{R}_launches_512.csv"}},
          open(f"{P}/ncu_traffic.json", "w"), indent=1)
# 2. full-set summary at 256^3
if os.path.exists(f"{G}/full256_{R}.ncu-rep"):
    s = subprocess.run([sys.executable, "scripts/ncu_summary.py", f"{G}/full256_{R}.ncu-rep"], capture_output=True, text=True).stdout
    s2 = subprocess.run([sys.executable, "scripts/ncu_source.py", f"{G}/full256_{R}.ncu-rep", "reorder_deposit", "15"], capture_output=True, text=True).stdout
    open(f"{P}/{R}_ncu_full_256.txt", "w").write(f"# {R}: ncu --set full, 256^3 x 8 ppc, step launches of reorder_deposit and push_key_brick\n" + s + "\n# top stall lines (reorder_deposit)\n" + s2)
for f in (f"bench_{R}.json", f"bench_ref_{R}.json", f"pytest_gpu_{R}.log", f"smoke_{R}.log", f"gpu_{R}.txt"):
    if os.path.exists(f"{G}/{f}"):
        txt = open(f"{G}/{f}").read()
        if f.startswith("pytest"):
            txt = "\n".join(txt.splitlines()[-15:]) + "\n"
        open(f"{P}/{R}_{f.replace('_' + R, '')}", "w").write(txt)
