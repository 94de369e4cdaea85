"""Per-role timeline of a forward GEMM (skip = 0 conv1, 1 conv2, 2 conv3, 3 fc, 4 heads).

    python tools/fwd_trace.py SKIP
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402
skip = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 2592
net = AtariNet(num_actions=6)
frames = torch.randint(0, 256, (n, 4, 84, 84), dtype=torch.uint8, device="cuda")
rew = torch.rand(n, device="cuda")
la = torch.randint(0, 6, (n,), device="cuda")
TT = 80
tr = torch.zeros(148 * TT * 16, dtype=torch.int64, device="cuda")
for it in range(3):
    if it == 2:
        N.lib().bp_gemm_trace_next(tr.data_ptr(), TT, skip)
    net._forward_kernels(frames, rew, la, repack=True, keep_x0=False)
torch.cuda.synchronize()
t = tr.view(148, TT, 16).cpu().numpy().astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
print(f"== forward gemm #{skip}: kernel span {np.nanmax(t[:, :, :8])/1e3:.1f} us, tiles on CTA 0: {int(np.sum(~np.isnan(t[0, :, 0])))}")
for name, a, bb in (("prod", 0, 1), ("mma", 2, 3), ("epi", 4, 5)):
    d = t[:, :, bb] - t[:, :, a]
    iv = t[:, 1:, a] - t[:, :-1, a]
    print(f"  {name}: median duration {np.nanmedian(d)/1e3:.3f} us, median start-to-start {np.nanmedian(iv)/1e3:.3f} us")
b = 0
for i in range(min(12, int(np.sum(~np.isnan(t[b, :, 0]))))):
    e = t[b, i]
    print(f"  tile {i:3d}: prod {e[0]/1e3:7.2f}-{e[1]/1e3:7.2f} mma {e[2]/1e3:7.2f}-{e[3]/1e3:7.2f}  epi {e[4]/1e3:7.2f}-{e[5]/1e3:7.2f} us")
