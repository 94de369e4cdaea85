"""Per-step phase timing of the LSTM recurrent kernels (CTA 0, %globaltimer)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from bench import make_batch  # noqa: E402
from paper_1910_03552_b200 import _native as N  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402

T1, B, A = 81, 32, 18
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N.check(N.lib().bp_lstm_set_mode(mode), "mode")
dev = torch.device("cuda")
net = AtariNet(num_actions=A, use_lstm=True)
batch = make_batch(T1 - 1, B, A, dev, 5)
n = T1 * B
tr = torch.zeros(2 * T1 * 4 + 2, dtype=torch.int64, device=dev)
st = net.initial_state(B)
lstm = dict(T1=T1, B=B, done=batch["done"].reshape(n).view(torch.uint8), h0=st[0], c0=st[1])
frames = batch["frame"].reshape(n, 4, 84, 84)
for it in range(3):
    if it == 2:
        N.check(N.lib().bp_lstm_trace(tr.data_ptr()), "trace")
    lg, bl = net._forward_kernels(frames, batch["reward"].reshape(n), batch["last_action"].reshape(n),
                                  repack=True, lstm=lstm)
    net._backward_kernels(torch.randn_like(lg), torch.randn_like(bl), batch["reward"].reshape(n),
                          batch["last_action"].reshape(n), net.flat_grads, lstm=lstm)
    torch.cuda.synchronize()
N.check(N.lib().bp_lstm_trace(None), "trace off")
tall = tr.cpu().double()
if mode == 2 or mode >= 16:  # cluster kernels record SM cycles: convert at the max SM clock
    tall = tall / 1.965
t = tall[:2 * T1 * 4].view(2, T1, 4)
print("forward set-up us", float(tall[-1] - tall[-2]) / 1e3)
f = t[0]
if mode == 1:
    fw = {"copy": f[1:, 1] - f[1:, 0], "compute": f[:, 2] - f[:, 1], "owner": f[:, 3] - f[:, 2],
          "barrier": f[1:, 0] - f[:-1, 3], "step": f[1:, 0] - f[:-1, 0]}
else:
    fw = {"mma": f[:-1, 1] - f[:-1, 0], "owner": f[:-1, 2] - f[:-1, 1], "exchange": f[:-1, 3] - f[:-1, 2],
          "step": f[1:-1, 0] - f[:-2, 0]}
print("forward (last layer) ns median:", {k: statistics.median(v.tolist()) for k, v in fw.items()},
      "total us", float(f[-1, 3] - f[0, 0]) / 1e3)
b = t[1]
# backward runs t = T1-1 .. 0
bw = {"partial": b[:-1, 1] - b[:-1, 0], "barrier": b[:-1, 2] - b[:-1, 1], "reduce+owner": b[:-1, 3] - b[:-1, 2],
      "step": b[:-1, 0] - b[1:, 0]}
print("backward (last layer) ns median:", {k: statistics.median(v.tolist()) for k, v in bw.items()},
      "total us", float(b[0, 3] - b[-1, 0]) / 1e3)
