"""One line per captured launch of an `ncu --page raw --csv` export (tools/ncu_export.sh): duration,
DRAM bytes and GB/s against the measured HBM peak, tensor (DMMA) pipe activity, issue activity,
achieved occupancy, L2 hit rate, instructions per warp.

Usage: python tools/ncu_summary.py <export.raw.csv> [...]   (writes to stdout)
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    HBM = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    HBM = 6558.7
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
          "second": 1.0}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def val(r, name, scale=None):
        if name not in ix:
            return float("nan")
        i = ix[name]
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            return float("nan")
        return v * (scale or {}).get(units[i], 1.0)

    print(f"# {os.path.basename(path)}  (HBM peak {HBM:.0f} GB/s)")
    for r in data:
        t = val(r, "gpu__time_duration.sum", TSCALE)
        rd, wr = val(r, "dram__bytes_read.sum", SCALE), val(r, "dram__bytes_write.sum", SCALE)
        nwarps = val(r, "launch__grid_size") * val(r, "launch__block_size") / 32.0
        inst = val(r, "smsp__inst_executed.sum")
        name = r[ix["Kernel Name"]].replace("h2b::", "")
        print(f"{name[:58]:58s} grid {r[ix['Grid Size']]:>16s} t={t * 1e3:8.3f} ms  DRAM {(rd + wr) / 1e9:7.2f} GB "
              f"= {(rd + wr) / t / 1e9:6.0f} GB/s ({(rd + wr) / t / 1e9 / HBM * 100:4.1f} % of peak)  "
              f"tensor {val(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):5.1f} %  "
              f"issue {val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f} %  "
              f"warps {val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} %  "
              f"L2 hit {val(r, 'lts__t_sector_hit_rate.pct'):5.1f} %  regs {val(r, 'launch__registers_per_thread'):.0f}  "
              f"inst/warp {inst / nwarps if nwarps else float('nan'):.0f}")


for p in sys.argv[1:]:
    main(p)
