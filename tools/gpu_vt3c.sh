python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
show() { python -c "
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['kernel'], d.get('T'), d.get('B'), d.get('A'), d.get('n'), round(d['median_s']*1e6,2), 'us', round(d['gbs']), 'GB/s', round(d['frac_of_hbm'],3))
" $1; }
timeout 300 python -m pytest tests/test_vtrace_gpu.py tests/test_learner_loss_gpu.py -q -x 2>&1 | tail -2
for bt in 0; do
BP_VT3_BT=$bt timeout 300 python -m paper_1910_03552_b200.kernel_bench --iters 20 > gpurun_out/kb_bt$bt.jsonl 2>&1; echo "BT=$bt"; show gpurun_out/kb_bt$bt.jsonl | grep -v rmsprop
BP_VT3_BT=$bt timeout 300 python -m pytest tests/test_vtrace_gpu.py tests/test_learner_loss_gpu.py -q -x 2>&1 | tail -1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vt3_kernel -o gpurun_out/vt3p_4096 -f python tools/vt_one.py 4096 > gpurun_out/ncu_full_vt3.log 2>&1; echo "ncu rc=$?"
