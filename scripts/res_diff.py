"""res_diff.py A.so B.so: kernels whose registers or stack (spill) bytes differ."""
import re
import subprocess
import sys


def res(so):
    out = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True, text=True).stdout
    d, fn = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and fn:
            d[fn] = (int(m.group(1)), int(m.group(2)))
            fn = None
    return d


a, b = res(sys.argv[1]), res(sys.argv[2])
for k in sorted(set(a) | set(b)):
    if a.get(k) != b.get(k):
        print(a.get(k), b.get(k), k[:160])
