python -m paper_1910_03552_b200.build > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -s 46 -c 23 --csv --log-file gpurun_out/launches_step.csv python tools/prof_step.py 3 > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.DictReader(open('gpurun_out/launches_step.csv')))
agg={}
for r in rows:
    k=(r['ID'], r['Kernel Name'][:60])
    agg.setdefault(k,{})[r['Metric Name']]=r['Metric Value']
tot=0
for (i,n),m in agg.items():
    t=float(m.get('gpu__time_duration.sum','0').replace(',',''))
    tot+=t
    print(f"{i:>4} {n:60s} {t:10.1f} ns  rd {m.get('dram__bytes_read.sum','')} wr {m.get('dram__bytes_write.sum','')} tc {m.get('sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed','')}")
print("total", tot)
PY
