# LSTM gx GEMM BN=64 vs 128 A/B (cfg3 kernel list, LSTM tests with the new setting)
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/gx
BP_GX_BN=1 timeout 600 python -m pytest tests/test_lstm_gpu.py tests/test_learn_parity_gpu.py -q -x 2>&1 | tail -2
for v in 0 1 0 1; do
  BP_GX_BN=$v timeout 300 python tools/graph_kernels.py 5 cfg3 > gpurun_out/gx/gk_cfg3_$v.txt 2>&1
  echo "gx_bn=$v"; grep -E "^  (6|11) |step span" gpurun_out/gx/gk_cfg3_$v.txt | cut -c1-110
done
