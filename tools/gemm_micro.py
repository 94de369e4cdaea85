"""Time the raw tcgen05 GEMM engine on AtariNet-like shapes (CUDA graphs, L2 flushed)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N
from paper_1910_03552_b200.kernel_bench import Timer

timer = Timer()
cases = [
    # name, M, N, K, a_mn, b_mn, splits, out_bf16
    ("conv2dgrad-like  KxMN bf16", 259200, 128, 256, 0, 1, 1, 1),
    ("conv2dgrad-like  KxK  bf16", 259200, 128, 256, 0, 0, 1, 1),
    ("conv1fwd-like    KxK  bf16", 1143040, 32, 256, 0, 0, 1, 1),
    ("conv2fwd-like    KxK  bf16", 259200, 64, 512, 0, 0, 1, 1),
    ("conv3fwd-like    KxK  bf16", 209920, 64, 576, 0, 0, 1, 1),
    ("fc-like          KxK  bf16", 2688, 512, 3136, 0, 0, 1, 1),
    ("conv3wgrad-like MNxMN f32 ", 640, 64, 209984, 1, 1, 30, 0),
    ("conv1wgrad-like MNxMN f32 ", 256, 32, 1143040, 1, 1, 74, 0),
    ("big square       KxK  bf16", 8192, 256, 8192, 0, 0, 1, 1),
]
for name, M, Nn, K, a_mn, b_mn, sp, ob in cases:
    A = torch.randn(M * K, device="cuda").to(torch.bfloat16)
    B = torch.randn(Nn * K, device="cuda").to(torch.bfloat16)
    m_pad = ((M + 127) // 128) * 128
    C = torch.empty(sp * m_pad * Nn, device="cuda", dtype=torch.bfloat16 if ob else torch.float32)
    fn = lambda: N.check(N.lib().bp_gemm_bf16_test(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, Nn, K,
                                                   a_mn, b_mn, sp, ob, N.stream_handle()), "gemm")
    r = timer.time(fn, iters=10, warmup=2)
    flops = 2.0 * M * Nn * K
    byts = (M * K + Nn * K) * 2 + sp * m_pad * Nn * (2 if ob else 4)
    print(f"{name}: {r['median_s']*1e6:8.1f} us  {flops/r['median_s']/1e12:7.1f} TFLOP/s  "
          f"{byts/r['median_s']/1e9:7.0f} GB/s (operand+output bytes)", flush=True)
