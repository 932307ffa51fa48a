"""Print the per-(phase, kernel) profile table of a tools/repro.py log with FP64 TFLOP/s."""
import ast
import sys

for path in sys.argv[1:]:
    print("==", path)
    for l in open(path).read().splitlines():
        if l.startswith("second run") or l.startswith("{'seg"):
            print(l)
        if l.startswith("{'name'"):
            e = ast.literal_eval(l)
            tf = 2 * e["macs"] / e["ms"] / 1e9 if e["macs"] else 0
            print(f"{e['name']:40s} {e['launches']:3d} {e['ms']:8.1f} ms {tf:6.1f} TF")
