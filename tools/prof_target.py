"""Tiny driver for ncu captures: runs one kernel config a few times.

    python tools/prof_target.py vtrace 80 4096 18
    python tools/prof_target.py loss 80 4096 18
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_03552_b200 import kernel_bench as kb  # noqa: E402

what, T, B, A = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
timer = kb.Timer()
if what == "vtrace":
    print(kb.bench_vtrace(T, B, A, timer, iters=3))
elif what == "loss":
    print(kb.bench_loss(T, B, A, timer, iters=3))
elif what == "rmsprop":
    print(kb.bench_rmsprop(T * B * A, timer, iters=3))
torch.cuda.synchronize()
