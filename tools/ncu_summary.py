"""Summarise an ncu report: key metrics + top stall source lines."""
import csv, subprocess, sys, io

rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return out
raw = list(csv.reader(io.StringIO(page("raw"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__t_bytes.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for h, u, v in zip(hdr, units, vals):
    if h in want or h.endswith("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"):
        print(f"{h:70s} {v:>16s} {u}")
src = list(csv.reader(io.StringIO(page("source", ["--print-source", "sass"]))))
# find header row
hi = next(i for i, r in enumerate(src) if "Source" in r)
H = src[hi]
i_s = H.index("Source"); i_w = H.index("Warp Stall Sampling (All Samples)")
rows = []
for r in src[hi + 1:]:
    try:
        rows.append((int(r[i_w] or 0), r[i_s][:100]))
    except Exception:
        pass
tot = sum(x[0] for x in rows) or 1
print("top stall samples (of", tot, ")")
for n, s in sorted(rows, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{n:6d} {100*n/tot:5.1f}%  {s}")
