python -m paper_1910_03552_b200.build > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/shift_trace.py
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['phase_seconds'])"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base function -k regex:"^(umma|vtrace|frames|pack|cast|finalize|sumsq|rmsprop|sample)" -s 42 -c 21 --csv --log-file gpurun_out/launches_step.csv python tools/prof_step.py 3 > gpurun_out/ncu_step.log 2>&1; echo "ncu rc=$?"
python tools/parse_launches.py gpurun_out/launches_step.csv
