python -m paper_1910_03552_b200.build > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/full_conv3_fwd python tools/prof_step.py 1 0 > /dev/null 2>&1; echo "rc=$?"
