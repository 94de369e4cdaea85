"""Window vs per-tap-box operand modes of the shifted GEMM (bp_gemm_shift_test), timed."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N  # noqa: E402
shapes = {"conv3": (2592 * 81, 64, 64, [dy * 9 + dx for dy in range(3) for dx in range(3)]),
          "conv2": (2592 * 100, 128, 64, [0, 1, 10, 11]),
          "conv1": (2592 * 441, 64, 32, [0, 1, 21, 22]),
          "aligned8": (2592 * 100, 128, 64, [0, 8, 16, 24])}
for name, (R, Cin, Nn, offs) in shapes.items():
    taps = len(offs)
    A = torch.randn(R, Cin, device="cuda").to(torch.bfloat16)
    B = (torch.randn(Nn, taps * Cin, device="cuda") * 0.1).to(torch.bfloat16)
    out = torch.empty(((R + 127) // 128 * 128, Nn), device="cuda")
    oc = (C.c_int * taps)(*offs)
    res = {}
    for mode in (0, 1):
        f = lambda: N.check(N.lib().bp_gemm_shift_test(A.data_ptr(), B.data_ptr(), out.data_ptr(), R, Cin, Nn,  # noqa
                                                       taps, oc, mode, None, 0, N.stream_handle()), "shift")
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        e1.synchronize()
        res[mode] = e0.elapsed_time(e1) / 10 * 1e3
    print(f"{name}: per-tap boxes {res[0]:.1f} us, window {res[1]:.1f} us")
