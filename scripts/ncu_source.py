"""Top SASS lines of one kernel of an ncu report by stall samples, with L1 traffic."""
import csv, io, subprocess, sys

def main(rep, kernel_regex, top=25):
    import re
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # sections: ["Kernel Name", name] then a header row starting with "Address"
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    sec = None
    for k, i in enumerate(starts):
        if re.search(kernel_regex, rows[i][1]):
            sec = rows[i + 1:(starts[k + 1] if k + 1 < len(starts) else len(rows))]
            break
    hdr = sec[0]; data = [r for r in sec[1:] if len(r) == len(hdr) and r[0] != "Address"]
    ix = {h: i for i, h in enumerate(hdr)}
    f = lambda r, k: float(r[ix[k]] or 0) if k in ix and r[ix[k]] not in ("", "-") else 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
    wf = sum(f(r, "L1 Wavefronts Shared") for r in data)
    l1g = sum(f(r, "L2 Theoretical Sectors Global") for r in data)
    print(f"samples {tot:.0f}  smem wavefronts {wf:.3g}  L2 sectors(global) {l1g:.3g}")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
        s = f(r, "Warp Stall Sampling (All Samples)")
        st = sorted(((f(r, h), h[6:]) for h in stalls), reverse=True)[:2]
        print(f"{100*s/tot:5.1f}% {r[ix['Source']][:58]:58s} smwf={f(r,'L1 Wavefronts Shared'):.2g} "
              f"L2sec={f(r,'L2 Theoretical Sectors Global'):.2g} {[(int(a),b) for a,b in st]}")

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
