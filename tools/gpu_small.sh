python -m paper_1910_03552_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_vtrace_gpu.py tests/test_learner_loss_gpu.py tests/test_learn_gpu.py tests/test_atari_gpu.py -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 28 -c 22 --csv python tools/prof_step.py 2 > gpurun_out/launch_small.csv 2>&1; python tools/parse_launches.py gpurun_out/launch_small.csv | head -24
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-200
