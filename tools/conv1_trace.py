"""Per-role timeline of the conv1 forward GEMM (u8 operand mode or bf16 grid mode).

    python tools/conv1_trace.py [u8=1]
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # 0 conv1, 1 conv2, 2 conv3, 3 fc, 4 heads
keep_x0 = not (len(sys.argv) > 3 and sys.argv[3] == "nox0")
N.lib().bp_atari_set_conv1_u8(mode)
n = int(sys.argv[4]) if len(sys.argv) > 4 else 2592
net = AtariNet(num_actions=6)
frames = torch.randint(0, 256, (n, 4, 84, 84), dtype=torch.uint8, device="cuda")
rew = torch.rand(n, device="cuda")
la = torch.randint(0, 6, (n,), device="cuda")
TT = 80
tr = torch.zeros(148 * TT * 16, dtype=torch.int64, device="cuda")
for it in range(3):
    if it == 2:
        N.lib().bp_gemm_trace_next(tr.data_ptr(), TT, skip)
    net._forward_kernels(frames, rew, la, repack=True, keep_x0=keep_x0)
torch.cuda.synchronize()
t = tr.view(148, TT, 16).cpu().numpy().astype(np.float64) / 1.965  # SM cycles -> ns at 1965 MHz
ntiles = [(n * 441 + 127) // 128, (n * 100 + 127) // 128, (n * 81 + 127) // 128,
          ((n + 127) // 128) * 8, (n + 127) // 128][skip]
per = [len(range(b, ntiles, 148)) for b in range(148)]
t = np.where(t > 0, t - t[:, :1, :1], np.nan)  # per-CTA clock origin
print(f"== gemm #{skip} u8={mode}: tiles/CTA {per[0]}, kernel span {np.nanmax(t)/1e3:.1f} us")
b = 0
for i in list(range(min(per[b], 6))) + list(range(max(6, min(per[b], TT) - 3), min(per[b], TT))):
    e = t[b, i]
    print(f"  tile {i:3d}: prod {e[0]/1e3:7.2f}-{e[1]/1e3:7.2f} conv {e[6]/1e3:7.2f}-{e[7]/1e3:7.2f} "
          f"mma {e[2]/1e3:7.2f}-{e[3]/1e3:7.2f}  epi {e[4]/1e3:7.2f}-{e[5]/1e3:7.2f} us")
for name, a, bb in (("prod", 0, 1), ("conv", 6, 7), ("conv-loop", 6, 8), ("conv-fence", 8, 9), ("mma", 2, 3), ("epi", 4, 5)):
    d = t[:, :, bb] - t[:, :, a]
    iv = t[:, 1:, a] - t[:, :-1, a]
    print(f"  {name}: median duration {np.nanmedian(d)/1e3:.3f} us, median start-to-start {np.nanmedian(iv)/1e3:.3f} us")
