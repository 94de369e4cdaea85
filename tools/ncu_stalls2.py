"""Top SASS lines of an ncu report with their dominant stall reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
H = rows[hi]
iS, iW = H.index("Source"), H.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in H if c.startswith("stall_") and "Not Issued" not in c]
data = []
for idx, r in enumerate(rows[hi + 1:]):
    try:
        w = int(r[iW] or 0)
    except ValueError:
        continue
    rs = sorted(((int(r[H.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:3]
    data.append((w, idx, r[iS].strip()[:70], rs))
tot = sum(d[0] for d in data) or 1
agg = {}
for d in data:
    for v, c in d[3]:
        pass
for c in reasons:
    agg[c[6:]] = sum(int(r[H.index(c)] or 0) for r in rows[hi + 1:] if len(r) == len(H))
print("total samples", tot, "by reason:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
for w, idx, src, rs in sorted(data, reverse=True)[:n]:
    print(f"{w:6d} {100*w/tot:5.1f}% #{idx:5d} {src:70s} {rs}")
