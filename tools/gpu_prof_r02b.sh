# round-2 profile set: conv1 forward full ncu (source) + bench launch list
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/r02
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 0 -c 1 -o gpurun_out/r02/full_conv1_fwd python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f1 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_wgrad -s 0 -c 1 -o gpurun_out/r02/full_conv1_wgrad python tools/prof_step.py 2 0 > /dev/null 2>&1; echo "f2 rc=$?"
ls -la gpurun_out/r02
