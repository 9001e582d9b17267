"""Compile libpic's sources with -Xptxas -v and print registers/spills/smem per kernel."""
import sys; sys.path.insert(0, ".")
import glob, re, subprocess, sys
srcs = sorted(glob.glob("paper_2605_05469_b200/csrc/*.cu"))
import paper_2605_05469_b200._build as B
inc, _ = B.nccl_dirs()
out = subprocess.run(["nvcc", "-I" + inc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
                      "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v", "-o", "/tmp/ptxas_probe.so", *srcs],
                     capture_output=True, text=True).stderr
name = None
for line in out.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        name = m.group(1)
        name = re.sub(r"_ZN3pic\d+_GLOBAL__N__\w+?_cu_[0-9a-f]+", "", name)[:60]
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = m.groups()
    m = re.search(r"Used (\d+) registers.*?(?:(\d+) bytes smem)?$", line)
    if m and name:
        print(f"{name:60s} regs={m.group(1):>3s} spill={spill} smem={m.group(2) or 0}")
        name = None
