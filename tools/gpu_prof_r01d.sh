# round-1 profile set v7 (final code of the round: + warp-split finalize, native infeed, stats pack)
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -c 90 --csv --log-file gpurun_out/launches_cfg1_v7.csv python tools/prof_step.py 3 0 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_v7.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:finalize -c 1 -o gpurun_out/full_finalize_v7 python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f1 rc=$?"
ls gpurun_out/
