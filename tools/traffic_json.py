"""profiles/rNN/traffic.json from an ncu launch list of the cfg1 learner step (dram bytes per
kernel): the forward (prep .. heads) and backward (pack_g .. finalize) phase sums of the last
complete step, plus per-launch V-trace / loss figures carried over from ncu --set full reports.

  python tools/traffic_json.py profiles/r02/launches_cfg1_step.csv profiles/r02/traffic.json \
      vtrace_from_logits_T80_B4096_A18=profiles/r02/ncu_full_vt3_4096.txt
"""
import collections
import csv
import json
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    hdr, data = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = data.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "m": {}})
        e["m"][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
    return data


def ncu_full_bytes(path):
    txt = open(path).read()
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(key + r"\s+([\d.,]+)\s+(\w+)", txt)
        tot += float(m.group(1).replace(",", "")) * UNIT[m.group(2)]
    return tot


def main():
    src, dst = sys.argv[1], sys.argv[2]
    data = launches(src)
    ids = sorted(data)
    preps = [i for i in ids if "prep_kernel" in data[i]["name"]]
    start = preps[-2]  # last complete step: the one before the final prep
    step = [i for i in ids if start <= i < preps[-1]]
    names = [data[i]["name"] for i in step]
    vt = next(k for k, n in enumerate(names) if "vt3_kernel" in n)
    pg = next(k for k, n in enumerate(names) if "pack_g_kernel" in n)
    fin = next(k for k, n in enumerate(names) if "finalize_kernel" in n)
    byt = lambda i: data[i]["m"]["dram__bytes_read.sum"] + data[i]["m"]["dram__bytes_write.sum"]  # noqa: E731
    fwd = step[:vt]
    bwd = step[pg:fin + 1]
    out = {"source": f"{src}: ncu launch list, last complete step (IDs {step[0]}-{step[-1]}); forward = "
                     "prep .. heads, backward = pack_g .. finalize; DRAM read + write bytes",
           "atari_forward_cfg1_step": sum(byt(i) for i in fwd),
           "atari_backward_cfg1_step": sum(byt(i) for i in bwd),
           "forward_kernels": [data[i]["name"][:60] for i in fwd],
           "backward_kernels": [data[i]["name"][:60] for i in bwd]}
    for kv in sys.argv[3:]:
        k, p = kv.split("=", 1)
        out[k] = ncu_full_bytes(p)
        out.setdefault("per_launch_sources", {})[k] = p
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if not isinstance(v, (list, dict))}, indent=1))


if __name__ == "__main__":
    main()
