"""Extract the per-launch DRAM traffic and key pipe metrics of an `ncu --set full` capture and
record them for bench.py's roofline.traffic (profiles/TRAFFIC.json).

Usage: python tools/ncu_traffic.py <report.ncu-rep> <key, e.g. cfg2:L9.targets/seg_gemm> [summary.txt]
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
out_txt = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def col(name):
    return hdr.index(name)


def val(r, name, scale=None):
    i = col(name)
    v = float(r[i]) if r[i] not in ("", "no data") else float("nan")
    return v * (scale or {}).get(units[i], 1.0)


METRICS = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
launches = []
for r in data:
    rd = val(r, "dram__bytes_read.sum", SCALE)
    wr = val(r, "dram__bytes_write.sum", SCALE)
    t = val(r, "gpu__time_duration.sum", TSCALE)
    e = {"kernel": r[col("Kernel Name")], "time_s": t, "dram_read": rd, "dram_write": wr,
         "dram_gbs": (rd + wr) / t / 1e9}
    for m in METRICS:
        e[m] = val(r, m)
    launches.append(e)
avg = sum(e["dram_read"] + e["dram_write"] for e in launches) / len(launches)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "TRAFFIC.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db[key] = {"dram_bytes_per_launch": avg, "launches_captured": len(launches),
           "source": f"ncu --set full ({os.path.basename(rep)}), dram__bytes_read.sum + dram__bytes_write.sum, "
                     f"mean over {len(launches)} captured launches"}
json.dump(db, open(path, "w"), indent=1)
lines = [f"# {rep} -> {key}"]
for e in launches:
    lines.append(f"{e['kernel'][:60]}  t={e['time_s'] * 1e3:.3f} ms  DRAM read {e['dram_read'] / 1e9:.2f} GB "
                 f"write {e['dram_write'] / 1e9:.2f} GB ({e['dram_gbs']:.0f} GB/s)")
    for m in METRICS:
        lines.append(f"    {m} = {e[m]:.3f}")
print("\n".join(lines))
if out_txt:
    open(out_txt, "w").write("\n".join(lines) + "\n")
