# inference tests + sampler/atari regressions + the inference bench leg
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_inference_gpu.py tests/test_atari_gpu.py tests/test_lstm_gpu.py -q -x > gpurun_out/pytest_inf.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_inf.log
timeout 300 python - > gpurun_out/inf_bench.log 2>&1 <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
from paper_1910_03552_b200.atari_net import AtariNet
from paper_1910_03552_b200 import kernel_bench
m = AtariNet(num_actions=6)
print(json.dumps(bench.bench_inference(m, 6, torch.device("cuda"), kernel_bench.Timer())))
PY
echo "inf rc=$?"; tail -3 gpurun_out/inf_bench.log
