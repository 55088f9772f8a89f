"""Print the sed expression that turns on FusedCfg's HS (and optionally TRIV)
option for every fused entry where it is legal (one FIR group, evenly split
tile), for A/B builds: python scripts/hs_variant.py [triv] [only=L:T,...]"""
import re
import sys

DEF = [None, None, None, None, 160, 96, 4, 2, 2, "false", 0, "false", "false"]
triv = "triv" in sys.argv
only = None
for a in sys.argv[1:]:
    if a.startswith("only="):
        only = {tuple(map(int, p.split(":"))) for p in a[5:].split(",")}
exprs = []
for f in ["tab_fused_main.cu", "tab_fused_small.cu", "tab_fused_fft.cu"]:
    for m in re.finditer(r"fused_entry<FusedCfg<([^>]*)>>", open("paper_1411_3656_b200/csrc/" + f).read()):
        args = [a.strip() for a in m.group(1).split(",")]
        full = args + [str(d) for d in DEF[len(args):]]
        L, T, RLOG = int(full[0]), int(full[1]), int(full[2])
        exact = full[3] == "true"
        wg = int(full[7])
        N = 1 << L
        ntg = N >> RLOG
        G = 256 // ntg if ntg <= 256 else 0
        B = max(1, (128 * wg * 16) // (N * max(G, 1)))
        tile_rows = max(G, 1) * B
        ok = T > 1 and not (len(full) > 11 and full[11] == 'true' and False) and tile_rows % wg == 0 and (only is None or (L, T) in only)
        if not ok:
            continue
        full[11] = "true"
        if triv and not exact and RLOG == 2 and T > 1:
            full[12] = "true"
        new = "fused_entry<FusedCfg<" + ", ".join(full) + ">>"
        exprs.append("s/" + m.group(0) + "/" + new + "/")
print(";".join(exprs))
