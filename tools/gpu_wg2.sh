python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_wgrad_window_gpu.py tests/test_conv1_u8_gpu.py -q -x > gpurun_out/pytest_wg.log 2>&1; echo "wg rc=$?"; tail -15 gpurun_out/pytest_wg.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 28 -c 26 --csv python tools/prof_step.py 1 > gpurun_out/launch_wg.csv 2>&1; echo "ncu rc=$?"
python tools/parse_launches.py gpurun_out/launch_wg.csv | head -30
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-700
