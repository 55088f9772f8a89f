"""Per-region stall breakdown from `ncu --page source --csv --print-source sass`.
Splits SASS at role boundaries given as address substrings (optional)."""
import csv
import collections
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_long_sb",
           "stall_math", "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected",
           "stall_short_sb", "stall_wait", "stall_membar", "stall_misc", "stall_sleep"]


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    data = rows[2:]
    f = lambda r, k: float(r[idx[k]] or 0)
    tot = collections.Counter()
    for r in data:
        for k in REASONS:
            if k in idx:
                tot[k] += f(r, k)
    s = sum(tot.values())
    print("total samples", s)
    for k, v in tot.most_common():
        print(f"  {k:26s} {v:9.0f} {100 * v / s:5.1f}%")
    print("top instructions:")
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
        rs = sorted(((f(r, k), k) for k in REASONS if k in idx), reverse=True)[:2]
        print(f'{r[idx["Address"]][-5:]} {f(r, "Warp Stall Sampling (All Samples)"):7.0f} '
              f'{rs[0][1][6:]}={rs[0][0]:.0f} {rs[1][1][6:]}={rs[1][0]:.0f}  '
              f'{r[idx["Source"]][:70]}')


if __name__ == "__main__":
    main(sys.argv[1])
