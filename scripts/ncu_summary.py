"""Summarise an ncu report: key SOL metrics, opcode mix, top stall lines."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout

det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Executed Instructions", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Eligible Warps Per Scheduler", "No Eligible", "Compute (SM) Throughput"]
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
if len(raw) >= 3:
    names, units, vals = raw[0], raw[1], raw[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
              "smsp__average_warp_latency_issue_stalled_barrier", "gpu__time_duration.sum"):
        for i, n in enumerate(names):
            if n == k:
                print(f"{k:60s} {vals[i]:>16s} {units[i]}")
sass = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hh = sass[1]; idx = {k: i for i, k in enumerate(hh)}
c = collections.Counter(); s = collections.Counter()
rows = sass[2:]
for r in rows:
    n = int(r[idx["Instructions Executed"]] or 0)
    op = re.sub(r"^@!?U?P\w+\s+", "", r[idx["Source"]].strip()).split(" ")[0]
    c[op] += n
    s[op] += int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(c.values())
print("total warp instructions", tot)
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {op:22s} {n:>12d} {100*n/tot:5.1f}%  stall-samples {s[op]}")
