"""Stall samples and executed instructions of one kernel aggregated by CUDA source line."""
import csv, subprocess, sys


def main(rep, kregex, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                          "-k", "regex:" + kregex], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    agg = {}
    for k, h in enumerate(hi):
        hdr = rows[h]
        end = hi[k + 1] - 3 if k + 1 < len(hi) else len(rows)
        ix = {n: i for i, n in enumerate(hdr)}
        cur = None
        for r in rows[h + 1:end]:
            if len(r) < len(hdr):
                continue
            if r[0]:
                cur = (int(r[0]), r[1].strip()[:88])
            if cur is None:
                continue

            def f(name):
                try:
                    return float(r[ix[name]] or 0)
                except (KeyError, ValueError):
                    return 0.0
            a = agg.setdefault(cur, [0.0, 0.0])
            a[0] += f("Warp Stall Sampling (All Samples)")
            a[1] += f("Instructions Executed")
        break   # first kernel section only
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"samples {ts:.0f} warp-instructions {ti:.3g}")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / ts:5.1f}% stall  {100 * v[1] / ti:5.1f}% inst  L{key[0]:<5d} {key[1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
