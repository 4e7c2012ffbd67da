"""Print SASS (address order) with exec counts and stall samples, filtered by min count."""
import csv, io, subprocess, sys
rep, lo = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}
for r in rows[2:]:
    n = int(r[idx["Instructions Executed"]] or 0)
    if n >= lo:
        print(f"{r[idx['Address']][-5:]} {n:>9d} {r[idx['Warp Stall Sampling (All Samples)']]:>5s}  {r[idx['Source']].strip()[:100]}")
