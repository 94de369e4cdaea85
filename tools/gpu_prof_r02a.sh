python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/r02
for w in cfg1 cfg3 inf1 inf1024 cfg4s; do
  timeout 300 python tools/graph_kernels.py 5 $w > gpurun_out/r02/graph_kernels_$w.txt 2>&1; echo "$w rc=$?"; tail -1 gpurun_out/r02/graph_kernels_$w.txt
done
timeout 300 python tools/graph_kernels.py 1 cfg4 > gpurun_out/r02/graph_kernels_cfg4.txt 2>&1; echo "cfg4 rc=$?"; tail -1 gpurun_out/r02/graph_kernels_cfg4.txt
timeout 300 python tools/lstm_trace.py 2 > gpurun_out/r02/lstm_trace.txt 2>&1; echo "trace rc=$?"; cat gpurun_out/r02/lstm_trace.txt | tail -4
