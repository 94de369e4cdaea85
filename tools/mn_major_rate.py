"""MMA throughput, K-major vs MN-major operands (bp_gemm_bf16_test), long-K split GEMMs."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N  # noqa: E402
for (M, Nn, K) in ((256, 64, 1 << 20), (640, 64, 1 << 18)):
    for amn, bmn in ((0, 0), (1, 1)):
        A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((K, Nn) if bmn else (Nn, K), device="cuda").to(torch.bfloat16)
        splits = 148 * 128 // M if M < 148 * 128 else 1
        splits = max(1, min(splits, K // 64))
        C = torch.empty((splits, (M + 127) // 128 * 128, Nn), device="cuda")
        f = lambda: N.check(N.lib().bp_gemm_bf16_test(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, Nn, K, amn, bmn,  # noqa
                                                      splits, 0, N.stream_handle()), "gemm")
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 5 * 1e-3
        print(f"M={M} N={Nn} K={K} a_mn={amn} b_mn={bmn} splits={splits}: {t*1e6:.1f} us, "
              f"{2*M*Nn*K/t/1e12:.1f} TFLOP/s, operand bytes {((M+Nn)*K*2)/t/1e9:.0f} GB/s")
