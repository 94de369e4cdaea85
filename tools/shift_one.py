import sys, ctypes as C
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N
R, Cin, Nn = 2592 * 81, 64, 64
offs = [dy * 9 + dx for dy in range(3) for dx in range(3)]
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
A = torch.randn(R, Cin, device="cuda").to(torch.bfloat16)
B = (torch.randn(Nn, 9 * Cin, device="cuda") * 0.1).to(torch.bfloat16)
out = torch.empty(((R + 127) // 128 * 128, Nn), device="cuda")
oc = (C.c_int * 9)(*offs)
for _ in range(3):
    N.check(N.lib().bp_gemm_shift_test(A.data_ptr(), B.data_ptr(), out.data_ptr(), R, Cin, Nn, 9, oc, mode,
                                       N.stream_handle()), "shift")
torch.cuda.synchronize()
