"""Shifted-tap GEMM: window modes vs per-tap boxes -- correctness vs torch + timing."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N
from paper_1910_03552_b200.kernel_bench import Timer
import ctypes as C

timer = Timer()
cases = [
    ("conv3-like", 2592 * 81, 64, 64, [dy * 9 + dx for dy in range(3) for dx in range(3)]),
    ("conv2-like", 2592 * 100, 128, 64, [0, 1, 10, 11]),
    ("conv1-like", 2592 * 441, 64, 32, [0, 1, 21, 22]),
    ("dgrad3-like", 2592 * 81, 64, 64, [-(dy * 9 + dx) for dy in range(3) for dx in range(3)]),
    ("small", 1000, 64, 64, [0, 3, 7, 13]),
]
for name, R, Cin, Nn, offs in cases:
    taps = len(offs)
    A = torch.randn(R, Cin, device="cuda").to(torch.bfloat16)
    B = (torch.randn(Nn, taps * Cin, device="cuda") * 0.1).to(torch.bfloat16)
    # reference: C[m] = sum_t A[m + off_t] . B[:, t]
    Af = A.float()
    ref = torch.zeros(R, Nn, device="cuda")
    for t, o in enumerate(offs):
        sh = torch.zeros_like(Af)
        lo, hi = max(0, -o), min(R, R - o)
        sh[lo:hi] = Af[lo + o:hi + o]
        ref += sh @ B[:, t * Cin:(t + 1) * Cin].float().t()
    offs_c = (C.c_int * taps)(*offs)
    for mode in (0, 1, 2):
        out = torch.full(((R + 127) // 128 * 128, Nn), float("nan"), device="cuda")
        fn = lambda: N.check(N.lib().bp_gemm_shift_test(A.data_ptr(), B.data_ptr(), out.data_ptr(), R, Cin, Nn,
                                                        taps, offs_c, mode, None, 0, N.stream_handle()), "shift")
        fn()
        torch.cuda.synchronize()
        err = float((out[:R] - ref).norm() / ref.norm())
        t = timer.time(fn, iters=10, warmup=2)["median_s"] if R > 100000 else float("nan")
        print(f"{name:12s} mode {mode}: rel err {err:.2e}   {t*1e6:8.1f} us", flush=True)
