"""make_traffic.py REP C T MODE N_SPECTRA_IN OUT.json [SUMMARY.txt]: the per-launch
DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernel in an
`ncu --set full` capture, keyed by configuration and kernel name for bench.py's
roofline.traffic (ncu_traffic matches the plan's kernel name against it)."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from scripts.ncu_summary import raw  # noqa: E402

rep, C, T, mode, S, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), sys.argv[6]
row = raw(rep)[0]


def val(k):
    v, u = row[k]
    v = float(v)
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3,
                "ns": 1e-6}.get(u, 1.0)


t = {"source": f"{rep} (ncu --set full --clock-control none, one launch of the bench's step)",
     "kernel": row["Kernel Name"][0], "n_channels": C, "n_taps": T, "mode": mode, "n_spectra_in": S,
     "dram_bytes_read": val("dram__bytes_read.sum"), "dram_bytes_write": val("dram__bytes_write.sum"),
     "gpu_time_ms_under_ncu": val("gpu__time_duration.sum")}
t["traffic_per_launch"] = t["dram_bytes_read"] + t["dram_bytes_write"]
t["algorithmic_bytes"] = 8 * C * (2 * S - T + 1)
t["traffic_over_algorithmic"] = t["traffic_per_launch"] / t["algorithmic_bytes"]
json.dump(t, open(out, "w"), indent=1)
print(json.dumps(t))
