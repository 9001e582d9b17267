"""Registers, stack frame and spills per kernel of the built libpic.so (cuobjdump -res-usage),
plus spill bytes from a -Xptxas -v compile with the same flags."""
import re
import subprocess
import sys

sys.path.insert(0, ".")
import paper_2605_05469_b200._build as B  # noqa: E402

lib = B.build_lib()
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
name = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = re.sub(r"_ZN3pic\d+_GLOBAL__N__\w+?_cu_[0-9a-f]+", "", m.group(1))[:64]
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and name:
        reg, stack, shared, local = m.groups()
        flag = "  <-- stack" if int(stack) > 0 else ""
        print(f"{name:64s} regs={reg:>3s} stack={stack:>4s} static_smem={shared:>5s}{flag}")
        name = None
