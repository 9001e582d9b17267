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
    elif r["Metric Name"].startswith("lts__t_requests"):
        d["l2_requests"] = v * {"request": 1, "Krequest": 1e3, "Mrequest": 1e6, "Grequest": 1e9}.get(unit, 1)
    elif r["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r["Metric Name"].split(".")[0].replace("dram__bytes_", "dram_")] = v * scale
out = sorted(launch.values(), key=lambda d: d["id"])
with open(f"{P}/{R}_launches_512.csv", "w") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "time_us", "dram_read_bytes", "dram_write_bytes", "l2_requests"])
    for d in out:
        w.writerow([d["id"], d["kernel"], d["grid"], d["block"], round(d.get("time_us", 0), 2),
                    int(d.get("dram_read", 0)), int(d.get("dram_write", 0)), int(d.get("l2_requests", 0))])
# per-kernel share of one step (cold-cache, serialised: compare shares); init-only
# launches (the push-less re-sort after the half kick) are left out
INIT_ONLY = ("k_reorder_deposit<0", "k_key_import", "k_sample", "k_half_kick")
agg = {}
for d in out:
    if d["kernel"].startswith(INIT_ONLY):
        continue
    a = agg.setdefault(d["kernel"], [0, 0.0, 0.0, 0.0])
    a[0] += 1; a[1] += d.get("time_us", 0); a[2] += d.get("dram_read", 0) + d.get("dram_write", 0)
    a[3] += d.get("l2_requests", 0)
tot = sum(a[1] for a in agg.values())
lines = [f"# {R}: ncu launch list, 512^3 x 8 ppc (bench config), gpu__time_duration + dram bytes, "
         f"--clock-control none; {len(out)} launches after skipping init",
         "kernel,launches,total_us,share,GB_per_launch,GBps,L2_requests_per_launch"]
for k, (n, t, b, q) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{n},{t:.1f},{t / tot:.3f},{b / n / 1e9:.3f},{b / (t * 1e-6) / 1e9 if t else 0:.0f},{q / n:.3e}")
open(f"{P}/{R}_launches_512_summary.csv", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
# 2. full-set captures at the bench config (512^3): summaries, hot source lines, and the
#    per-launch DRAM traffic bench.py reports for the dominant kernel
tr = {k: (b / n) for k, (n, t, b, q) in agg.items()}
full = {}
for rep, kernels in ((f"{G}/full512_{R}.ncu-rep", ("reorder_deposit", "push_key_brick")),
                     (f"{G}/full512fft_{R}.ncu-rep", ("fft_z_mul", "fft_x_inv", "place"))):
    if not os.path.exists(rep):
        continue
    s = subprocess.run([sys.executable, "scripts/ncu_summary.py", rep], capture_output=True, text=True).stdout
    for m in re.finditer(r"raw (?:void )?(?:unnamed>::)?(k_\w+)[^{]*(\{[^}]*\})", s):
        d = eval(m.group(2))
        full.setdefault(m.group(1), (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * 1e9)
    hot = ""
    for k in kernels:
        hot += f"\n# hot source lines: {k}\n" + subprocess.run(
            [sys.executable, "scripts/ncu_lines.py", rep, k, "14"], capture_output=True, text=True).stdout
    tag = os.path.basename(rep).replace(".ncu-rep", "").replace(f"_{R}", "")
    tag = {"full512": f"{R}_ncu_full_512", "full512fft": f"{R}_ncu_full_512_fft_place"}[tag]
    open(f"{P}/{tag}.txt", "w").write(f"# {R}: ncu --set full --clock-control none, 512^3 x 8 ppc bench step launches\n"
                                      + s + hot)
traffic = {"reorder_deposit": full.get("k_reorder_deposit", tr.get("k_reorder_deposit")),
           "push_key": full.get("k_push_key_brick", tr.get("k_push_key_brick")),
           "source": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                     f"(profiles/{R}_ncu_full_512.txt); launch list profiles/{R}_launches_512.csv"}
try:
    allt = json.load(open(f"{P}/ncu_traffic.json"))
except Exception:
    allt = {}
allt["landau3d_512^3x8ppc_fft"] = traffic            # the other configs' entries are kept
json.dump(allt, open(f"{P}/ncu_traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
