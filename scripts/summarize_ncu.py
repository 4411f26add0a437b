"""Summarise ncu outputs into the committed profiles/ directory.

    python scripts/summarize_ncu.py launches <launches.csv> <out.md> [--last-block N]
    python scripts/summarize_ncu.py full <prof.ncu-rep> <out.md>

``launches``: per-kernel count, total and mean duration and share of the
launch list (cold-cache, serialised -- compare shares, not absolutes); with
--last-block N only the last N launches (one steady block) are summarised.
``full``: the headline metrics of each captured launch (duration, DRAM bytes,
tensor / MUFU / FMA pipe utilisation, issue, occupancy, registers).
"""

from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys


def _kname(k: str) -> str:
    k = re.sub(r"\(.*", "", k.replace("void ", ""))
    return k.replace("lp::", "")


def launches(path: str, out: str, last: int | None) -> None:
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = [r for r in csv.DictReader(io.StringIO(text)) if r["Metric Name"] == "gpu__time_duration.sum"]
    if last:
        rows = rows[-last:]
    agg = collections.OrderedDict()
    for r in rows:
        k = _kname(r["Kernel Name"]) + " grid" + r["Grid Size"]
        ns = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1.0)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list: {path}", "",
             f"{len(rows)} launches, {tot / 1e6:.3f} ms total (cold-cache, serialised; compare shares)", "",
             "| kernel (grid) | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {ns / tot:.3f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU/MUFU pipe % (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % (active)"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe % (active)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]


def full(path: str, out: str) -> dict:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {path}", ""]
    res = {}
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        name = _kname(rec.get("Kernel Name", "?"))
        lines += [f"## {name} (launch id {rec.get('ID')})", "", "| metric | value |", "|---|---|"]
        vals = {}
        for key, label in METRICS:
            if key in rec:
                u = units[hdr.index(key)]
                lines.append(f"| {label} (`{key}`) | {rec[key]} {u} |")
                vals[key] = (rec[key], u)
        try:
            rd = float(vals["dram__bytes_read.sum"][0]) * _scale(vals["dram__bytes_read.sum"][1])
            wr = float(vals["dram__bytes_write.sum"][0]) * _scale(vals["dram__bytes_write.sum"][1])
            lines.append(f"| DRAM traffic read+write | {(rd + wr) / 1e6:.1f} MB |")
            res.setdefault(name, []).append(rd + wr)
        except (KeyError, ValueError):
            pass
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return res


def _scale(u: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        last = None
        if "--last-block" in sys.argv:
            last = int(sys.argv[sys.argv.index("--last-block") + 1])
        launches(sys.argv[2], sys.argv[3], last)
    else:
        r = full(sys.argv[2], sys.argv[3])
        if len(sys.argv) > 4:
            json.dump(r, open(sys.argv[4], "w"), indent=1)
