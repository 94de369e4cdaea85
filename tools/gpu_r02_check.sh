# quick validation of the current code: GPU tests, smoke, bench
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/chk
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/chk/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/chk/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/chk/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/chk/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/chk/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/chk/bench.log | cut -c1-600
