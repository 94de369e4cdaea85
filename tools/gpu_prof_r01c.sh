# round-1 profile set v6 (3 epilogue warpgroups + compile-time epilogue kinds, PDL, column-sum
# warps for db1/db2, stats written straight to pinned memory)
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -c 90 --csv --log-file gpurun_out/launches_cfg1_v6.csv python tools/prof_step.py 3 0 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 300 ncu --metrics $M --clock-control none -s 60 -c 80 --csv --log-file gpurun_out/launches_cfg3_v6.csv python tools/prof_step.py 3 1 > /dev/null 2>&1; echo "ncu3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_v6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 0 -c 1 -o gpurun_out/full_conv1_fwd_v6 python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f1 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 8 -c 1 -o gpurun_out/full_conv2_dgrad_v6 python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f2 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_wgrad -s 0 -c 1 -o gpurun_out/full_conv1_wgrad_v6 python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f3 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vt3_kernel -c 2 -o gpurun_out/full_vt3_4096_v6 python tools/vt_one.py 4096 > /dev/null 2>&1; echo "f4 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vt3_kernel -c 2 -o gpurun_out/full_vt3_65536_v6 python tools/vt_one.py 65536 > /dev/null 2>&1; echo "f5 rc=$?"
python tools/graph_kernels.py 10 > gpurun_out/graph_kernels_v6.txt 2>&1; echo "graph rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v6.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_v6.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v6.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_v6.log | cut -c1-300
ls gpurun_out/
