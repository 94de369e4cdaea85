python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
show() { python -c "
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['kernel'], d.get('T'), d.get('B'), d.get('A'), d.get('n'), round(d['median_s']*1e6,2), 'us', round(d['gbs']), 'GB/s', round(d['frac_of_hbm'],3))
" $1; }
for impl in 3 2; do
BP_VTRACE_IMPL=$impl timeout 300 python -m paper_1910_03552_b200.kernel_bench --iters 30 > gpurun_out/kbench_$impl.jsonl 2>&1; echo "kbench impl=$impl rc=$?"; show gpurun_out/kbench_$impl.jsonl
done
for impl in 3 2; do
BP_VTRACE_IMPL=$impl timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/vt_one.py 4096 > gpurun_out/ncu_vt_$impl.csv 2>&1; echo "ncu impl=$impl rc=$?"
grep -E "vt[23]_kernel" gpurun_out/ncu_vt_$impl.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
done
