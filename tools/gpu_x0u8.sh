# u8 X0 A/B: parity tests, then the cfg1 / cfg4-shard kernel lists and the bench with X0 u8 on / off
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/x0
timeout 600 python -m pytest tests/test_conv1_u8_gpu.py tests/test_learn_parity_gpu.py tests/test_wgrad_window_gpu.py -q -x > gpurun_out/x0/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/x0/pytest.log
for v in 1 0; do
  BP_X0_U8=$v timeout 300 python tools/graph_kernels.py 5 cfg1 > gpurun_out/x0/gk_cfg1_$v.txt 2>&1
  BP_X0_U8=$v timeout 300 python tools/graph_kernels.py 2 cfg4s > gpurun_out/x0/gk_cfg4s_$v.txt 2>&1
  BP_X0_U8=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/x0/bench_$v.log 2>&1
  echo "x0u8=$v"; grep -E "wgrad_win_kernel<32|umma_gemm_kernel<32, 0, 0, 128, true, 1, 1|step span" gpurun_out/x0/gk_cfg1_$v.txt | cut -c1-100
  grep -E "wgrad_win_kernel<32|umma_gemm_kernel<32, 0, 0, 128, true, 1, 1|step span" gpurun_out/x0/gk_cfg4s_$v.txt | cut -c1-100
  tail -1 gpurun_out/x0/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d.get('cfg4',{}).get('ms_per_step'))"
done
