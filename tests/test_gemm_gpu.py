"""The raw tcgen05 GEMM engine (bp_gemm_bf16_test) against torch fp32 matmul of
the same bf16 operands: every operand-major / swizzle / tile-width / split-K
combination the AtariNet kernels use.  Tolerance: fp32-accumulation order only
(relative L2 <= 1e-5, max-abs <= 1e-4 * max|ref|)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(M, N, K, a_mn, b_mn, splits=1, seed=0):
    from paper_1910_03552_b200 import _native as Nt

    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    a_store = A.t().contiguous() if a_mn else A.contiguous()
    b_store = B.t().contiguous() if b_mn else B.contiguous()
    m_pad = ((M + 127) // 128) * 128
    C = torch.full((splits, m_pad, N), float("nan"), device="cuda")
    Nt.check(Nt.lib().bp_gemm_bf16_test(a_store.data_ptr(), b_store.data_ptr(), C.data_ptr(), M, N, K,
                                        int(a_mn), int(b_mn), splits, 0, Nt.stream_handle()),
             "bp_gemm_bf16_test")
    torch.cuda.synchronize()
    got = C.sum(0)[:M]
    ref = A.float() @ B.float().t()
    return got, ref


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,splits", [
    (128, 32, 64, 0, 0, 1),
    (256, 32, 256, 0, 0, 1),
    (384, 64, 512, 0, 0, 1),
    (256, 128, 256, 0, 0, 1),
    (256, 256, 3136 // 49 * 49, 0, 0, 1),
    (1024, 512, 576, 0, 0, 1),
    (256, 32, 1024, 1, 1, 1),
    (256, 32, 4096, 1, 1, 7),
    (512, 64, 1024, 1, 1, 3),
    (640, 512, 640, 1, 1, 2),
    (256, 64, 512, 0, 1, 1),
    (384, 128, 576, 0, 1, 1),
    (256, 64, 512, 1, 0, 1),
])
def test_engine_matches_torch(M, N, K, a_mn, b_mn, splits):
    got, ref = _run(M, N, K, a_mn, b_mn, splits)
    assert torch.isfinite(got).all()
    err = (got - ref).norm() / ref.norm()
    assert err < 1e-5, f"rel L2 {err}"
    assert (got - ref).abs().max() <= 1e-4 * ref.abs().max()
