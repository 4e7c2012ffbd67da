import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out))); n, u, v = r[0], r[1], r[2]
items = [(n[i], v[i]) for i in range(len(n)) if "smsp__average_warps_issue_stalled" in n[i] and n[i].endswith("_per_issue_active.ratio")]
for k, val in sorted(items, key=lambda x: -float(x[1] or 0))[:12]:
    print(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {float(val):.3f}")
