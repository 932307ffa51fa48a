"""Summarise an ncu launch list (gpu__time_duration.sum per launch, kernels renamed by their
NVTX phase range, tools/gpu_round.sh) into per-phase / per-kernel shares.

Usage: python tools/launch_summary.py gpurun_out/launches_cfg2.csv [top]
ncu serialises launches and runs them cold, so compare SHARES, not absolute times."""
import collections
import csv
import re
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
data = [r for r in rows[start + 1:] if len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum"]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ni = next(i for i, h in enumerate(hdr) if "Push/Pop_Range" in h)


def phase(r):
    m = re.search(r'<default domain>:([^:"]+):([^:"]+)', r[ni])
    if m:
        return m.group(1) + ":" + m.group(2)
    return "(outside the product: input constructor) " + re.sub(r"\(.*", "", r[ki])[:60]


tot, cnt = collections.Counter(), collections.Counter()
for r in data:
    p = phase(r)
    tot[p] += float(r[vi])
    cnt[p] += 1
all_ns = sum(tot.values())
print(f"# {path}: {len(data)} launches, {all_ns / 1e6:.1f} ms serialised device time")
print(f"{'ms':>10} {'share':>7} {'launches':>9}  phase:kernel")
for k, v in tot.most_common(top):
    print(f"{v / 1e6:10.2f} {v / all_ns:7.1%} {cnt[k]:9d}  {k}")
