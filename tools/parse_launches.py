import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
agg = {}
order = []
for r in rows:
    k = r['ID']
    if k not in agg:
        agg[k] = {'name': r['Kernel Name'], 'grid': r['Grid Size'], 'block': r['Block Size']}
        order.append(k)
    agg[k][r['Metric Name']] = r['Metric Value']
tot = 0
for k in order:
    m = agg[k]
    t = float(m.get('gpu__time_duration.sum', '0').replace(',', ''))
    tot += t
    rd = float(m.get('dram__bytes_read.sum', '0').replace(',', '')) / 1e6
    wr = float(m.get('dram__bytes_write.sum', '0').replace(',', '')) / 1e6
    tc = m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', m.get('sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed', ''))
    print(f"{k:>4} {m['name'][:70]:70s} {m['grid']:>14s} {t/1e3:9.1f} us  rd {rd:8.1f} MB wr {wr:8.1f} MB tc {tc}")
print("total us", tot / 1e3)
