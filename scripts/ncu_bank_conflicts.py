#!/usr/bin/env python
"""Shared-memory bank conflicts of an ncu --set full --import-source on
report, attributed per SASS instruction and per CUDA source line:
instructions executed, shared wavefronts, ideal wavefronts, excessive.
Usage: python scripts/ncu_bank_conflicts.py REPORT [min_excessive]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 1


def page(what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # the first row may be a kernel/file banner; the header has "Source"
    hi = next(i for i, r in enumerate(rows) if "Source" in r)
    return rows[hi], rows[hi + 1:]


def num(r, idx, k):
    try:
        return int(float(r[idx[k]] or 0))
    except (KeyError, ValueError):
        return 0


for what in ("sass", "cuda"):
    h, rows = page(what)
    idx = {k: i for i, k in enumerate(h)}
    cols = [k for k in h if "Shared" in k or "Conflict" in k]
    if what == "sass":
        print("columns:", cols)
    wf = next((k for k in h if k.startswith("L1 Wavefronts Shared") and "Ideal" not in k
               and "Excessive" not in k), None)
    ideal = next((k for k in h if k.startswith("L1 Wavefronts Shared Ideal")), None)
    exc = next((k for k in h if k.startswith("L1 Wavefronts Shared Excessive")), None)
    tot_w = tot_i = tot_e = 0
    print(f"== {what}: lines with >= {lo} excessive shared wavefronts")
    for r in rows:
        e = num(r, idx, exc) if exc else 0
        w = num(r, idx, wf) if wf else 0
        i = num(r, idx, ideal) if ideal else 0
        tot_w += w
        tot_i += i
        tot_e += e
        if e >= lo:
            loc = r[idx["Address"]][-5:] if what == "sass" else r[idx.get("#", 0)]
            print(f"{loc:>6} exec={num(r, idx, 'Instructions Executed'):>11d} wavefronts={w:>11d} "
                  f"ideal={i:>11d} excessive={e:>11d}  {r[idx['Source']].strip()[:90]}")
    print(f"totals ({what}): wavefronts={tot_w} ideal={tot_i} excessive={tot_e}")
