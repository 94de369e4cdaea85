"""Per-kernel key metrics of an ncu report (multi-kernel safe) + top stall lines of kernel 0.

    python tools/ncu_summary2.py REPORT [TOP]
"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
hdr, units = raw[0], raw[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for row in raw[2:]:
    d = dict(zip(hdr, row))
    print("kernel:", d.get("Kernel Name", "?")[:110])
    for k in want:
        if k in d:
            u = units[hdr.index(k)]
            print(f"  {k:95s} {d[k]:>14s} {u}")
print()
out = subprocess.run([sys.executable, "tools/ncu_stalls2.py", rep, str(top), "0"], capture_output=True, text=True)
print("top stall SASS lines (kernel 0):")
print(out.stdout)
