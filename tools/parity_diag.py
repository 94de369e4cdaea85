"""Where do the GPU network and the bf16-emulating oracle diverge?  Per storage point:
fraction of bf16 elements that differ and the relative L2 of the difference (GPU forward on
cuda:0 vs oracle.atari_ref.emulated_* in fp64 on the same device)."""
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from oracle import atari_ref  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def main(T=20, B=8, A=18):
    torch.manual_seed(11)
    ref = atari_ref.AtariNetRef(num_actions=A)
    with torch.no_grad():
        for p in ref.parameters():
            p.add_(0.05 * torch.randn_like(p))
    net = AtariNet(num_actions=A)
    net.load_state_dict(ref.state_dict())
    batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(T, B, A, seed=40).items()}
    n = (T + 1) * B
    logits, base = net._forward_kernels(batch["frame"].reshape(n, 4, 84, 84), batch["reward"].reshape(n),
                                        batch["last_action"].reshape(n), repack=True)
    torch.cuda.synchronize()
    t = net._bufs.t
    x1 = t["x1"][: n * 100].float().view(n, 10, 10, 2, 2, 32).permute(0, 5, 1, 3, 2, 4).reshape(n, 32, 20, 20)
    x2 = t["x2"][: n * 81].float().view(n, 9, 9, 64).permute(0, 3, 1, 2)
    x3 = t["x3"][:n].float().view(n, 7, 7, 64).permute(0, 3, 1, 2)
    core = t["core"][:n, :513 + A].float()
    r64 = ref.double().cuda()
    st = atari_ref.st_bf16
    with torch.no_grad():
        x = batch["frame"].reshape(n, 4, 84, 84).double()
        z1 = F.conv2d(x, st(r64.conv1.weight), None, stride=4) / 255.0 + r64.conv1.bias[:, None, None]
        a1 = atari_ref.bf16_round(F.relu(z1))
        print("X1 (from exact input)  differ %.5f rel %.2e" % ((a1 != x1.double()).float().mean(), rel(x1, a1)))
        # each layer from the GPU's OWN previous activation: per-layer kernel error only
        z2 = F.conv2d(x1.double(), st(r64.conv2.weight), r64.conv2.bias, stride=2)
        a2 = atari_ref.bf16_round(F.relu(z2))
        print("X2 (from GPU X1)       differ %.5f rel %.2e" % ((a2 != x2.double()).float().mean(), rel(x2, a2)))
        z3 = F.conv2d(x2.double(), st(r64.conv3.weight), r64.conv3.bias)
        a3 = atari_ref.bf16_round(F.relu(z3))
        print("X3 (from GPU X2)       differ %.5f rel %.2e" % ((a3 != x3.double()).float().mean(), rel(x3, a3)))
        zf = x3.double().reshape(n, -1) @ st(r64.fc.weight).t() + r64.fc.bias
        af = atari_ref.bf16_round(F.relu(zf))
        print("fc (from GPU X3)       differ %.5f rel %.2e" % ((af != core[:, :512].double()).float().mean(),
                                                            rel(core[:, :512], af)))
        # pre-activation accuracy where no rounding hides it: f32 pre-act of fc vs the f64 one
        lg = core.double() @ st(r64.policy.weight).t() + st(r64.policy.bias)
        print("logits (from GPU core) rel %.2e" % rel(logits, lg))
        # whole chain
        out, _ = atari_ref.emulated_forward(r64, {k: v for k, v in batch.items()})
        print("logits end-to-end      rel %.2e" % rel(logits.view(T + 1, B, A), out["policy_logits"]))
        # z-precision of the GPU tensor cores: fc pre-activation reconstructed from relu outputs
        pos = af > 0
        zgpu = core[:, :512].double()
        d = ((zgpu - zf).abs() / zf.abs().clamp_min(1e-30))[pos & (zgpu > 0)]
        print("fc: |bf16(gpu) - z64|/|z64| median %.2e (bf16 half-ulp ~2e-3)" % d.median())




def gemm_precision(M=1024, N=512, K=3136):
    """Relative error of the tcgen05 engine vs fp64 for zero-mean and all-positive operands
    (truncating accumulation shows up as a K-proportional bias on positive data)."""
    from paper_1910_03552_b200 import _native as Nt

    for kind in ("randn", "positive"):
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.randn(M, K, device="cuda", generator=g)
        B = torch.randn(N, K, device="cuda", generator=g)
        if kind == "positive":
            A, B = A.abs(), B.abs()
        A, B = A.to(torch.bfloat16), B.to(torch.bfloat16)
        C = torch.zeros(1, M, N, device="cuda")
        Nt.check(Nt.lib().bp_gemm_bf16_test(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, 0, 1, 0,
                                            Nt.stream_handle()), "gemm")
        ref = A.double() @ B.double().t()
        f32 = (A.float() @ B.float().t()).double()
        print("gemm %s K=%d: engine rel %.2e  mean signed %.2e | cublas f32 rel %.2e" % (
            kind, K, rel(C[0], ref), float(((C[0].double() - ref) / ref.abs().clamp_min(1e-30)).mean()),
            rel(f32, ref)))


if __name__ == "__main__":
    torch.backends.cuda.matmul.allow_tf32 = False
    gemm_precision()
    gemm_precision(K=576)
    main(*[int(a) for a in sys.argv[1:]])
