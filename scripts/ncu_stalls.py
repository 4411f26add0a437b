"""Top warp-stall reasons and instructions of one kernel in an ncu report
(source page, SASS).  python scripts/ncu_stalls.py <rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, k):
    try:
        return int(r[ix[k]] or 0)
    except (ValueError, IndexError):
        return 0


tot = {s: sum(num(r, s) for r in data) for s in stalls}
alls = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
print("samples", alls)
for s, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {s:28s} {v:8d} {100 * v / max(alls, 1):5.1f}%")
for i, r in enumerate(data):
    r.append(i)
for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top_n]:
    n = num(r, "Warp Stall Sampling (All Samples)")
    main = max(stalls, key=lambda s: num(r, s))
    print(f"{r[-1]:5d} {n:7d} {main:24s} {r[1][:90]}")
