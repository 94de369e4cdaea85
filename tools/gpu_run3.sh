python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 240 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo "gemm rc=$?"
tail -25 gpurun_out/pytest_gemm.log
timeout 300 python -m pytest tests/test_vtrace_gpu.py tests/test_learner_loss_gpu.py tests/test_optim_gpu.py -x -q > gpurun_out/pytest_vt.log 2>&1; echo "vt rc=$?"
tail -5 gpurun_out/pytest_vt.log
timeout 300 python -m pytest tests/test_atari_gpu.py -q > gpurun_out/pytest_atari.log 2>&1; echo "atari rc=$?"
tail -40 gpurun_out/pytest_atari.log
timeout 300 python -m pytest tests/test_learn_gpu.py -q > gpurun_out/pytest_learn.log 2>&1; echo "learn rc=$?"
tail -30 gpurun_out/pytest_learn.log
timeout 300 python -m paper_1910_03552_b200.kernel_bench --quick --iters 20 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"
cat gpurun_out/kbench.jsonl
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench.log
