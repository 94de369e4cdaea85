import sys, torch
sys.path.insert(0, ".")
from paper_1910_03552_b200 import learner_ops as lo
T, B, A = 80, 4096, 18
g = torch.Generator(device="cuda").manual_seed(0)
logits = torch.randn(T, B, A, device="cuda", generator=g)
baseline = torch.randn(T + 1, B, device="cuda", generator=g)
beh = torch.randn(T, B, A, device="cuda", generator=g)
act = torch.randint(0, A, (T, B), device="cuda", generator=g)
rew = torch.rand(T, B, device="cuda", generator=g)
done = torch.rand(T, B, device="cuda", generator=g) < 0.05
ll = lo.LearnerLoss()
dl, db, losses = ll(logits, baseline, beh, act, rew, done, lo.VtraceConfig())
torch.cuda.synchronize()
print(losses)
