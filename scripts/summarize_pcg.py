"""Summaries of the PCG (BJ config 5) ncu outputs in gpurun_out/ -> profiles/ (per round)."""
import csv, io, json, os, subprocess, sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
G, P = "gpurun_out", "profiles"


def short(kn):
    depth, cut = 0, len(kn)
    for i in range(len(kn) - 1, -1, -1):      # strip the trailing (parameter list)
        depth += kn[i] == ")"
        depth -= kn[i] == "("
        if depth == 0:
            cut = i
            break
    return kn[:cut].replace("unnamed>::", "").replace("void ", "")


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
rows = [l for l in open(f"{G}/launches_pcg512_{R}.csv") if l.startswith('"')]
launch = {}
for r in csv.DictReader(io.StringIO("".join(rows))):
    d = launch.setdefault(int(r["ID"]), {"id": int(r["ID"]), "kernel": short(r["Kernel Name"])})
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        d["time_us"] = v * TSCALE.get(r["Metric Unit"], 1.0)
    elif r["Metric Name"].startswith("dram__bytes"):
        d[r["Metric Name"].split(".")[0]] = v * SCALE.get(r["Metric Unit"], 1)
out = sorted(launch.values(), key=lambda d: d["id"])
with open(f"{P}/{R}_launches_pcg512.csv", "w") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "time_us", "dram_read_bytes", "dram_write_bytes"])
    for d in out:
        w.writerow([d["id"], d["kernel"], round(d.get("time_us", 0), 2), int(d.get("dram__bytes_read", 0)),
                    int(d.get("dram__bytes_write", 0))])
agg = {}
for d in out:
    a = agg.setdefault(d["kernel"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("time_us", 0)
    a[2] += d.get("dram__bytes_read", 0) + d.get("dram__bytes_write", 0)
tot = sum(a[1] for a in agg.values())
lines = [f"# {R}: ncu launch window of the 512^3 x 8 ppc PCG step (BJ config 5), gpu__time_duration + dram "
         f"bytes, --clock-control none; {len(out)} consecutive launches inside a step (CG iterations)",
         "kernel,launches,total_us,share,GB_per_launch,GBps"]
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{n},{t:.1f},{t / tot:.3f},{b / n / 1e9:.3f},{b / (t * 1e-6) / 1e9 if t else 0:.0f}")
open(f"{P}/{R}_launches_pcg512_summary.csv", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

rep = f"{G}/full_pcg512_{R}.ncu-rep"
txt = subprocess.run([sys.executable, "scripts/ncu_summary.py", rep], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = {x: i for i, x in enumerate(rr[0])}
per = {}
txt += "\n# per-launch DRAM bytes (base units)\n"
for r in rr[2:]:
    k = short(r[h["Kernel Name"]])
    b = float(r[h["dram__bytes_read.sum"]]) + float(r[h["dram__bytes_write.sum"]])
    per.setdefault(k, b)
    txt += f"{k}: read {float(r[h['dram__bytes_read.sum']]):.4g} B, write {float(r[h['dram__bytes_write.sum']]):.4g} B, " \
           f"{float(r[h['gpu__time_duration.sum']]):.4g} ns\n"
open(f"{P}/{R}_ncu_full_pcg512.txt", "w").write(f"# {R}: ncu --set full --clock-control none, 512^3 x 8 ppc PCG step\n" + txt)
print(txt)
tj = json.load(open(f"{P}/ncu_traffic.json")) if os.path.exists(f"{P}/ncu_traffic.json") else {}
sor = next((v for k, v in per.items() if k.startswith("k_sor4<0, false")), None) or \
      next((v for k, v in per.items() if k.startswith("k_sor4")), None)
tj["landau3d_512^3x8ppc_pcg"] = {"pcg_ssor": sor, "source": f"dram__bytes_read.sum + dram__bytes_write.sum per "
                                 f"k_sor4 half-sweep launch, ncu --set full (profiles/{R}_ncu_full_pcg512.txt)"}
json.dump(tj, open(f"{P}/ncu_traffic.json", "w"), indent=1)
