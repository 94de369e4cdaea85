"""One from_logits / learner-loss launch at T=80 A=18 and the given B (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import kernel_bench as kb, learner_ops as lo, vtrace  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
x = kb._vtrace_inputs(80, B, 18, 0)
vtrace.from_logits(*x)
f = kb._loss_call(80, B, 18, 0, lo.LearnerLoss(), lo.VtraceConfig())
f()
torch.cuda.synchronize()
