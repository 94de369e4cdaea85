python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -m paper_1910_03552_b200.kernel_bench --iters 30 > gpurun_out/kbench.jsonl 2> gpurun_out/kbench.err; echo "kbench rc=$?"
cat gpurun_out/kbench.jsonl; tail -5 gpurun_out/kbench.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vtrace_kernel -s 6 -c 1 -o gpurun_out/prof_vtrace2 python tools/prof_target.py vtrace 80 4096 18 > gpurun_out/ncu_vtrace.log 2>&1; echo "ncu rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vtrace_kernel -s 6 -c 1 -o gpurun_out/prof_loss2 python tools/prof_target.py loss 80 4096 18 > gpurun_out/ncu_loss.log 2>&1; echo "ncu rc=$?"
