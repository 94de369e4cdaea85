"""Per-role timeline of the shifted GEMM (conv-like shapes)."""
import sys, ctypes as C
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import _native as N
shapes = {"conv3": (2592 * 81, 64, 64, [dy * 9 + dx for dy in range(3) for dx in range(3)]),
          "conv1": (2592 * 441, 64, 32, [0, 1, 21, 22]),
          "conv2": (2592 * 100, 128, 64, [0, 1, 10, 11])}
for name, (R, Cin, Nn, offs) in shapes.items():
    taps = len(offs)
    A = torch.randn(R, Cin, device="cuda").to(torch.bfloat16)
    B = (torch.randn(Nn, taps * Cin, device="cuda") * 0.1).to(torch.bfloat16)
    out = torch.empty(((R + 127) // 128 * 128, Nn), device="cuda")
    oc = (C.c_int * taps)(*offs)
    TT = 80
    tr = torch.zeros(148 * TT * 8, dtype=torch.int64, device="cuda")
    for it in range(3):
        N.check(N.lib().bp_gemm_shift_test(A.data_ptr(), B.data_ptr(), out.data_ptr(), R, Cin, Nn, taps, oc, 1,
                                           tr.data_ptr(), TT, N.stream_handle()), "shift")
    torch.cuda.synchronize()
    t = tr.view(148, TT, 8).cpu().numpy().astype(np.float64)
    ntiles = (R + 127) // 128
    per = [len(range(b, ntiles, 148)) for b in range(148)]
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, np.nan)
    b = 0
    print(f"== {name}: tiles/CTA {per[0]}, kernel span {np.nanmax(t)/1e3:.1f} us")
    for i in list(range(min(per[b], 6))) + list(range(max(6, per[b] - 3), per[b])):
        e = t[b, i]
        print(f"  tile {i:3d}: prod {e[0]/1e3:7.2f}-{e[1]/1e3:7.2f}  mma {e[2]/1e3:7.2f}-{e[3]/1e3:7.2f}  epi {e[4]/1e3:7.2f}-{e[5]/1e3:7.2f} us")
    d = t[:, 1:, 4] - t[:, :-1, 4]
    print(f"  median epi-to-epi interval {np.nanmedian(d)/1e3:.2f} us; median epi duration "
          f"{np.nanmedian(t[:, :, 5] - t[:, :, 4])/1e3:.2f} us; median mma span {np.nanmedian(t[:, :, 3]-t[:, :, 2])/1e3:.2f} us; "
          f"median (mma start - prod start) {np.nanmedian(t[:, :, 2]-t[:, :, 0])/1e3:.2f} us")
