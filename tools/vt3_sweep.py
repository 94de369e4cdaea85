"""Sweep the tile-resident V-trace / loss kernel's tile width (BP_VT3_BT) and CTAs per SM
(BP_VT3_CTAS_PER_SM) at the large-batch sizes; one subprocess per setting (the knobs are
read once per process).  Prints one JSON line per (setting, kernel, B)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1910_03552_b200 import kernel_bench as kb

    timer = kb.Timer()
    peak, _ = kb._peaks()
    for B in (4096, 16384):
        for r in (kb.bench_vtrace(80, B, 18, timer, 40), kb.bench_loss(80, B, 18, timer, 40)):
            print(json.dumps(dict(bt=os.environ.get("BP_VT3_BT", "auto"),
                                  cps=os.environ.get("BP_VT3_CTAS_PER_SM", "max"), kernel=r["kernel"], B=B,
                                  us=round(r["median_s"] * 1e6, 2), frac=round(r["gbs"] / peak, 3))), flush=True)
    sys.exit(0)

for bt in ("0", "2", "4", "8"):
    for cps in ("0", "1", "2", "3", "4"):
        env = dict(os.environ, BP_VT3_BT=bt, BP_VT3_CTAS_PER_SM=cps)
        if bt == "0":
            env.pop("BP_VT3_BT")
        if cps == "0":
            env.pop("BP_VT3_CTAS_PER_SM")
        out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True,
                             timeout=300)
        sys.stdout.write(out.stdout or out.stderr[-400:])
        sys.stdout.flush()
