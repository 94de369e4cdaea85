python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_vtrace_gpu.py tests/test_learner_loss_gpu.py tests/test_learn_gpu.py -q -x > gpurun_out/pytest_vt.log 2>&1; echo "vt rc=$?"; tail -15 gpurun_out/pytest_vt.log
for impl in 3 2; do
BP_VTRACE_IMPL=$impl timeout 300 python -m paper_1910_03552_b200.kernel_bench --iters 30 > gpurun_out/kbench_$impl.jsonl 2>&1; echo "kbench impl=$impl rc=$?"
python -c "
import json
for l in open('gpurun_out/kbench_$impl.jsonl'):
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['kernel'], d.get('T'), d.get('B'), d.get('A'), d.get('n'), round(d['median_s']*1e6,1), 'us', round(d['gbs']), 'GB/s', round(d['frac_of_hbm'],3))
"
done
