python -m paper_1910_03552_b200.build > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lstm_cl_fwd -c 1 -o gpurun_out/full_lstm_cl_fwd python tools/prof_step.py 1 1 > /dev/null 2>&1; echo "rc=$?"
