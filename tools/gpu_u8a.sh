python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_conv1_u8_gpu.py -q -x > gpurun_out/pytest_u8.log 2>&1; echo "u8 rc=$?"; tail -3 gpurun_out/pytest_u8.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 28 -c 6 --csv python tools/prof_step.py 1 > gpurun_out/launch_u8.csv 2>&1; echo "ncu rc=$?"
python tools/parse_launches.py gpurun_out/launch_u8.csv | head -30
timeout 600 ncu --set full --import-source on --clock-control none -k regex:umma_gemm_kernel --launch-skip 0 -c 1 -o gpurun_out/conv1_u8 -f python tools/prof_step.py 1 > gpurun_out/ncu_conv1_u8.log 2>&1; echo "ncu full rc=$?"
