"""Top SASS lines of an ncu report with their dominant stall reasons.

    python tools/ncu_stalls2.py REPORT [N] [KERNEL_INDEX]
"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
heads = [i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r]
hi = heads[kidx]
end = heads[kidx + 1] if kidx + 1 < len(heads) else len(rows)
H = rows[hi]
body = [r for r in rows[hi + 1:end] if len(r) == len(H)]
iS, iW = H.index("Source"), H.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in H if c.startswith("stall_") and "Not Issued" not in c]
num = lambda x: int(float(x)) if x not in ("", None) else 0  # noqa: E731
data = []
for idx, r in enumerate(body):
    w = num(r[iW])
    rs = sorted(((num(r[H.index(c)]), c[6:]) for c in reasons), reverse=True)[:3]
    data.append((w, idx, r[iS].strip()[:70], rs))
tot = sum(d[0] for d in data) or 1
agg = {c[6:]: sum(num(r[H.index(c)]) for r in body) for c in reasons}
print("total samples", tot, "by reason:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
for w, idx, src, rs in sorted(data, reverse=True)[:n]:
    print(f"{w:6d} {100*w/tot:5.1f}% #{idx:5d} {src:70s} {rs}")
