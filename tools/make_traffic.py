"""profiles/rNN/traffic.json from a round's ncu captures: DRAM read+write bytes per step of the
AtariNet forward / backward kernel groups (from the eager cfg1 step launch list) and per launch
of the V-trace / fused-loss kernels (from their --set full reports).

    python tools/make_traffic.py OUT_JSON STEP_CSV [NAME=REPORT.ncu-rep[@KERNEL_INDEX] ...]
"""
import csv
import json
import subprocess
import sys

out, step_csv = sys.argv[1], sys.argv[2]
lines = open(step_csv).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
agg, order = {}, []
for r in rows:
    k = r["ID"]
    if k not in agg:
        agg[k] = {"name": r["Kernel Name"]}
        order.append(k)
    agg[k][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
names = [agg[k]["name"] for k in order]
preps = [i for i, n in enumerate(names) if "prep_kernel" in n]
a, b = preps[-2], preps[-1]  # the last complete step
step = order[a:b]
fwd, bwd, in_bwd = [], [], False
for k in step:
    n = agg[k]["name"]
    if "vt3_kernel" in n:
        in_bwd = True
        continue
    if any(x in n for x in ("sumsq", "rmsprop", "pack_stats", "Fill", "elementwise")):
        continue
    (bwd if in_bwd else fwd).append(k)
tb = lambda ks: sum(agg[k].get("dram__bytes_read.sum", 0) + agg[k].get("dram__bytes_write.sum", 0) for k in ks)
res = {"source": f"ncu launch list {step_csv} (last complete eager step) + --set full reports",
       "atari_forward_cfg1_step": tb(fwd), "atari_backward_cfg1_step": tb(bwd),
       "forward_kernels": [agg[k]["name"][:60] for k in fwd],
       "backward_kernels": [agg[k]["name"][:60] for k in bwd]}
for arg in sys.argv[3:]:
    name, rep = arg.split("=", 1)
    idx = -1
    if "@" in rep:
        rep, idx = rep.split("@")
        idx = int(idx)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rr = list(csv.reader(txt.splitlines()))
    h = rr[0]
    vals = []
    for r in rr[2:]:
        d = dict(zip(h, r))
        def num(key):
            v = d.get(key, "0").replace(",", "")
            return float(v) if v else 0.0
        vals.append(num("dram__bytes_read.sum") + num("dram__bytes_write.sum"))
    if vals:
        res[name] = vals[idx]
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if not isinstance(v, list)}, indent=1))
