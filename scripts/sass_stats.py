"""Per-kernel SASS stats from cuobjdump: max register index, instruction count,
MOV count and the Blackwell-specific opcodes (UBLKCP, FFMA2/FMUL2/FADD2, DFMA,
SYNCS, USETMAXREG) — the evidence the kernels use the sm_100a features."""
import collections
import re
import subprocess
import sys

so = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur = None
stats = collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        stats[cur] = collections.Counter()
        continue
    if cur is None or "/*" not in line:
        continue
    ins = line.split("*/", 1)[1].strip() if "*/" in line else ""
    if not ins or ins.startswith("/*"):
        continue
    s = stats[cur]
    s["insts"] += 1
    op = ins.split()[0]
    if op.startswith("@"):
        op = ins.split()[1]
    base = op.split(".")[0].rstrip(";")
    for key in ("MOV", "UBLKCP", "FFMA2", "FMUL2", "FADD2", "DFMA", "DMUL", "SYNCS", "USETMAXREG",
                "LDS", "STS", "STG", "LDG", "BAR"):
        if base == key:
            s[key] += 1
    for r in re.findall(r"\bR(\d+)\b", ins):
        s["maxreg"] = max(s["maxreg"], int(r) + 1)
for name, s in stats.items():
    if pat in name:
        short = re.sub(r"_ZN4ppfg", "", name)[:70]
        print(short, dict(s))
