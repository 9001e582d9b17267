"""Summarise an ncu report: key metrics per kernel + top stall lines (source page)."""
import csv, io, subprocess, sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"]

def main(rep, top=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
    cur = None
    for r in rows[1:]:
        k = r[ix["Kernel Name"]][:70] + " #" + r[ix["ID"]]
        if k != cur:
            cur = k; print("==", k)
        if r[ix["Metric Name"]] in KEYS:
            print("   %-40s %10s %s" % (r[ix["Metric Name"]], r[ix["Metric Value"]], r[ix["Metric Unit"]]))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]; ixr = {x: i for i, x in enumerate(h)}
    for r in rr[2:]:
        name = r[ixr["Kernel Name"]][:60]
        vals = {m: r[ixr[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum") if m in ixr}
        print("raw", name, vals)

if __name__ == "__main__":
    main(sys.argv[1])
