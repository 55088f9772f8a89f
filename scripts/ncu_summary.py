"""Summarise an ncu --set full report for the judge/profiles: SOL, issue,
occupancy, stall reasons, DRAM bytes, smem wavefronts, instruction counts."""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    rows = []
    for v in r[2:]:
        rows.append({n: (val, un) for n, un, val in zip(h, u, v)})
    return rows


KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg",
        "smsp__cycles_active.avg"]


def main(rep):
    for row in raw(rep):
        for k in KEYS:
            if k in row:
                print(f"{k:60s} {row[k][0]} {row[k][1]}")
        stalls = [(k, float(v[0])) for k, v in row.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and
                  k.endswith("_per_issue_active.ratio") and v[0] not in ("", "n/a")]
        stalls.sort(key=lambda x: -x[1])
        print("stall reasons (warps per issue):")
        for k, v in stalls[:10]:
            print(f"  {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:.3f}")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
