import sys, torch
sys.path.insert(0, ".")
from oracle import atari_ref
from paper_1910_03552_b200.atari_net import AtariNet
torch.manual_seed(3)
A = 18
ref = atari_ref.AtariNetRef(num_actions=A)
with torch.no_grad():
    for p in ref.parameters():
        p.add_(0.05 * torch.randn_like(p))
net = AtariNet(num_actions=A)
net.load_state_dict(ref.state_dict())
b = atari_ref.synthetic_batch(0, 256, A, seed=5)
o = {k: v[0].cuda() for k, v in b.items()}
with torch.no_grad():
    want = ref({k: v[None] for k, v in b.items() if k in ("frame", "reward", "last_action")} | {"frame": b["frame"][:1]})[0]["policy_logits"][0]
for k in (256, 1, 2, 8, 32, 100, 256):
    for x0 in (True, False):
        lg, _ = net._forward_kernels(o["frame"][:k].contiguous(), o["reward"][:k].contiguous(), o["last_action"][:k].contiguous(), keep_x0=x0, repack=True)
        torch.cuda.synchronize()
        e = (lg.cpu() - want[:k]).norm() / want[:k].norm()
        print(k, x0, float(e), lg[0, :4].tolist(), want[0, :4].tolist())
