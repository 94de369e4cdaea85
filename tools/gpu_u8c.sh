python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:umma_gemm_kernel --launch-skip 0 -c 1 -o gpurun_out/conv1_u8 -f python tools/prof_step.py 1 > gpurun_out/ncu_conv1_u8.log 2>&1; echo "ncu full rc=$?"
