"""Aggregate an `ncu --metrics gpu__time_duration.sum,... --csv` launch list by kernel."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; idx = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in rows[1:]:
    k = r[idx["Kernel Name"]].split("(")[0][-44:]; m = r[idx["Metric Name"]]
    v = float(r[idx["Metric Value"]].replace(",", ""))
    agg[k][m] += v
    if m == "gpu__time_duration.sum":
        cnt[k] += 1
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"{'kernel':46s} {'launches':>8s} {'time ms':>9s} {'share':>6s} {'dram rd GB':>10s} {'dram wr GB':>10s} {'L2 GB':>7s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    print(f"{k:46s} {cnt[k]:8d} {a['gpu__time_duration.sum']/1e6:9.2f} {100*a['gpu__time_duration.sum']/tot:5.1f}% "
          f"{a.get('dram__bytes_read.sum',0)/1e9:10.2f} {a.get('dram__bytes_write.sum',0)/1e9:10.2f} {a.get('lts__t_bytes.sum',0)/1e9:7.1f}")
