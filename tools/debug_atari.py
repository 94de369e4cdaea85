"""Compare every AtariNet intermediate (activations, pre-activation gradients,
parameter gradients) of the GPU kernels against autograd on the torch-CPU oracle."""
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from oracle import atari_ref  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402


def rel(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


T, B, A = int(sys.argv[1]) if len(sys.argv) > 1 else 2, 3, 6
torch.manual_seed(3)
ref = atari_ref.AtariNetRef(num_actions=A)
with torch.no_grad():
    for p in ref.parameters():
        p.add_(0.05 * torch.randn_like(p))
net = AtariNet(num_actions=A)
net.load_state_dict(ref.state_dict())
batch = atari_ref.synthetic_batch(T, B, A, seed=2)
n = (T + 1) * B
g = torch.Generator().manual_seed(5)
dl = torch.randn(n, A, generator=g)
db = torch.randn(n, generator=g)

# oracle with retained intermediates
x = batch["frame"].reshape(n, 4, 84, 84).float() / 255.0
z1 = ref.conv1(x); z1.retain_grad(); a1 = F.relu(z1)
z2 = ref.conv2(a1); z2.retain_grad(); a2 = F.relu(z2)
z3 = ref.conv3(a2); z3.retain_grad(); a3 = F.relu(z3)
zf = ref.fc(a3.reshape(n, -1)); zf.retain_grad(); h = F.relu(zf)
core = torch.cat([h, torch.clamp(batch["reward"].reshape(n, 1), -1, 1),
                  F.one_hot(batch["last_action"].reshape(n), A).float()], -1)
logits = ref.policy(core)
base = ref.baseline(core).reshape(n)
torch.autograd.backward([logits, base], [dl, db])

cb = {k: v.cuda() for k, v in batch.items()}
lg, bs = net._forward_kernels(cb["frame"].reshape(n, 4, 84, 84), cb["reward"].reshape(n),
                              cb["last_action"].reshape(n))
grads = torch.full_like(net.flat_params, float("nan"))
net._backward_kernels(dl.cuda(), db.cuda(), cb["reward"].reshape(n), cb["last_action"].reshape(n), grads)
torch.cuda.synchronize()
t = net._bufs.t
print("logits", rel(lg, logits), "baseline", rel(bs, base))
# X1: s2d of a1 [n,10,10,(py,px,c)]
x1 = t["x1"][: n * 100].float().cpu().view(n, 10, 10, 2, 2, 32)
a1_g = x1.permute(0, 5, 1, 3, 2, 4).reshape(n, 32, 20, 20)
print("a1", rel(a1_g, a1))
a2_g = t["x2"][: n * 81].float().cpu().view(n, 9, 9, 64).permute(0, 3, 1, 2)
print("a2", rel(a2_g, a2))
a3_g = t["x3"][:n].float().cpu().view(n, 7, 7, 64).permute(0, 3, 1, 2)
print("a3", rel(a3_g, a3))
print("h", rel(t["core"][:n, :512].float().cpu(), h))
print("d_fc", rel(t["d_fc"][:n].float().cpu(), zf.grad))
d3 = t["d_pre3"][: n * 81].float().cpu().view(n, 9, 9, 64)
print("d_pre3", rel(d3[:, :7, :7].permute(0, 3, 1, 2), z3.grad),
      "pad max", float(d3[:, 7:].abs().max()), float(d3[:, :, 7:].abs().max()))
d2 = t["d_pre2"][: n * 100].float().cpu().view(n, 10, 10, 64)
print("d_pre2", rel(d2[:, :9, :9].permute(0, 3, 1, 2), z2.grad),
      "pad max", float(d2[:, 9:].abs().max()), float(d2[:, :, 9:].abs().max()))
d1 = t["d_pre1"][: n * 441].float().cpu().view(n, 21, 21, 32)
print("d_pre1", rel(d1[:, :20, :20].permute(0, 3, 1, 2), z1.grad),
      "pad max", float(d1[:, 20:].abs().max()), float(d1[:, :, 20:].abs().max()))
tg = net.torch_layout_grads(grads)
for k, p in ref.named_parameters():
    print(k, rel(tg[k], p.grad))
