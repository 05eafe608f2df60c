"""Summarise an .ncu-rep: key SOL metrics, stall reasons, top stalled SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = det[0]
iN, iV, iU, iS = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Section Name")
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Issue Slots Busy", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
for r in det[1:]:
    if r[iN] in want:
        print(f"{r[iN]:40s} {r[iV]} {r[iU]}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
names, vals = raw[0], raw[2]
d = dict(zip(names, vals))
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__inst_executed_pipe_fp64.sum",
          "sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
          "smsp__inst_executed.sum", "sass__inst_executed_local_loads", "sass__inst_executed_local_stores"]:
    print(f"{k:60s} {d.get(k)} {raw[1][names.index(k)] if k in names else ''}")
st = [(n[len('smsp__pcsamp_warps_issue_stalled_'):], float(v.replace(',', '') or 0)) for n, v in d.items()
      if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{n} {v / tot * 100:.1f}%" for n, v in sorted(st, key=lambda t: -t[1])[:10]))
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv"]))))
hdr = src[1]
S = hdr.index("Warp Stall Sampling (All Samples)")
cols = [(k, n) for k, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
rows = []
for r in src[2:]:
    try:
        rows.append((float(r[S]), r))
    except Exception:
        pass
tot = sum(x for x, _ in rows) or 1
for s, r in sorted(rows, key=lambda t: -t[0])[:top]:
    rs = sorted([(float(r[k] or 0), n[6:]) for k, n in cols], reverse=True)[:2]
    print(f"{s / tot * 100:5.2f}% {r[0][-5:]} {r[1].strip()[:58]:58s} {rs[0][1]} {rs[1][1]}")
