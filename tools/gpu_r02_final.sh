# round-2 validation + profile set on the current code
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02/bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02/bench_ref.log | cut -c1-200
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -c 90 --csv --log-file gpurun_out/r02/launches_cfg1_step.csv python tools/prof_step.py 3 0 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 300 ncu --metrics $M --clock-control none -s 80 -c 90 --csv --log-file gpurun_out/r02/launches_cfg3_step.csv python tools/prof_step.py 3 1 > /dev/null 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lstm_cl_fwd -c 1 -o gpurun_out/r02/full_lstm_fwd python tools/prof_step.py 1 1 > /dev/null 2>&1; echo "f lstm rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vt3_kernel -c 2 -o gpurun_out/r02/full_vt3_4096 python tools/vt_one.py 4096 > /dev/null 2>&1; echo "f vt3 rc=$?"
for w in cfg1 cfg3 inf1 inf1024 cfg4s; do timeout 300 python tools/graph_kernels.py 5 $w > gpurun_out/r02/graph_kernels_$w.txt 2>&1; done; timeout 300 python tools/graph_kernels.py 1 cfg4 > gpurun_out/r02/graph_kernels_cfg4.txt 2>&1; echo graphs done
ls gpurun_out/r02
