python -m paper_1910_03552_b200.build > /dev/null 2>&1 || exit 1
timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:umma_gemm_kernel<\(int\)128' -s 1 -c 1 -o gpurun_out/prof_conv2dgrad2 python tools/prof_step.py 3 > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
