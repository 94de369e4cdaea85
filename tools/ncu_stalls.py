"""Per-stall-reason totals and top SASS lines of an ncu report (excluding idle-warp EXIT/barrier)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
H = rows[hi]
i_s = H.index("Source")
reasons = [h for h in H if h.startswith("stall_") and "Not Issued" not in h]
idx = {r: H.index(r) for r in reasons}
tot = {r: 0 for r in reasons}
lines = []
for r in rows[hi + 1:]:
    src = r[i_s]
    if "EXIT" in src or "WARPSYNC.ALL" in src or "BAR.SYNC" in src:
        continue
    vals = {k: int(r[i] or 0) for k, i in idx.items()}
    for k, v in vals.items():
        tot[k] += v
    lines.append((sum(vals.values()), src[:90], max(vals, key=vals.get)))
T = sum(tot.values()) or 1
print("stall totals (excluding idle EXIT/WARPSYNC/BAR lines):")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {v:7d} {100*v/T:5.1f}%")
print("top lines:")
for n, s, why in sorted(lines, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{n:6d} {why:18s} {s}")
