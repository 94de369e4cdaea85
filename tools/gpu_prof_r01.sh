# round-1 profile set: launch lists (one learner step, both configs) + full captures
set -x
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
# step 1 of prof_step is the warm-up (first pack); profile the launches of step 2
timeout 300 ncu --metrics $M --clock-control none -s 22 -c 22 --csv --log-file gpurun_out/launches_cfg1.csv python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 300 ncu --metrics $M --clock-control none -s 38 -c 40 --csv --log-file gpurun_out/launches_cfg3.csv python tools/prof_step.py 2 1 > /dev/null 2>&1; echo "ncu3 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu bench rc=$?"
# full captures of the top kernels
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 14 -c 1 -o gpurun_out/full_conv1_fwd python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f1 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 22 -c 1 -o gpurun_out/full_conv2_dgrad python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f2 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 23 -c 1 -o gpurun_out/full_conv1_wgrad python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f3 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vt2_kernel -s 3 -c 1 -o gpurun_out/full_vtrace_4096 python tools/prof_target.py vtrace 80 4096 18 > /dev/null 2>&1; echo "f4 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vt2_kernel -s 3 -c 1 -o gpurun_out/full_vtrace_65536 python tools/prof_target.py vtrace 80 65536 18 > /dev/null 2>&1; echo "f5 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vt2_kernel -s 3 -c 1 -o gpurun_out/full_loss_4096 python tools/prof_target.py loss 80 4096 18 > /dev/null 2>&1; echo "f6 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lstm_fwd -s 2 -c 1 -o gpurun_out/full_lstm_fwd python tools/prof_step.py 2 1 > /dev/null 2>&1; echo "f7 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lstm_bwd -s 2 -c 1 -o gpurun_out/full_lstm_bwd python tools/prof_step.py 2 1 > /dev/null 2>&1; echo "f8 rc=$?"
ls -la gpurun_out/
