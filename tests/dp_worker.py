"""Worker for the data-parallel tests (spawned with torch.multiprocessing)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def oracle_dp(rank, world, port, out_q):
    """CPU oracle: shard-gradient SUM over gloo == full-batch gradient."""
    from oracle import atari_ref

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    model = atari_ref.AtariNetRef(num_actions=4)
    T, B = 3, 4
    batch = atari_ref.synthetic_batch(T, B, 4, seed=7)
    lo, hi = rank * B // world, (rank + 1) * B // world
    shard = {k: v[:, lo:hi].contiguous() for k, v in batch.items()}
    flags = dict(atari_ref.DEFAULT_FLAGS)
    total, _, _ = atari_ref.learn_losses(model, shard, flags)
    total.backward()
    flat = torch.cat([p.grad.reshape(-1) for p in model.parameters()])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    tot = total.detach().clone()
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    if rank == 0:
        model.zero_grad()
        full_total, _, _ = atari_ref.learn_losses(model, batch, flags)
        full_total.backward()
        full = torch.cat([p.grad.reshape(-1) for p in model.parameters()])
        out_q.put((float((flat - full).norm() / full.norm()), float(tot), float(full_total)))
    dist.destroy_process_group()


def fused_dp(rank, world, port, out_q, backend="gloo"):
    """GPU: FusedLearner(process_group) on B/world columns per rank.  gloo: every rank on cuda:0;
    nccl: rank r on cuda:r (needs >= world GPUs).  Reports the PRE-optimiser flat gradients
    (all-reduced) and the first update against a single-process run on the full batch."""
    from oracle import atari_ref
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    T, B, A = 10, 8, 6
    flags = dict(atari_ref.DEFAULT_FLAGS)
    batch = {k: v.to(dev) for k, v in atari_ref.synthetic_batch(T, B, A, seed=3).items()}
    lo, hi = rank * B // world, (rank + 1) * B // world
    shard = {k: v[:, lo:hi].contiguous() for k, v in batch.items()}
    torch.manual_seed(5)
    net = AtariNet(num_actions=A, device=dev)
    opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
    p0 = net.flat_params.clone()
    L = learner.FusedLearner(net, flags, T, B // world, process_group=True)
    # 1. no optimiser: the all-reduced flat gradient (graph replays on NCCL: eager, capture, replay)
    for _ in range(3):
        losses = L.step(shard, None).clone()
    torch.cuda.synchronize()
    grads = net.flat_grads.clone().cpu()
    # 2. one step with the fused clip + RMSProp
    L.step(shard, opt)
    torch.cuda.synchronize()
    upd = (net.flat_params - p0).cpu()
    gathered = [torch.zeros_like(upd) for _ in range(world)]
    if backend == "nccl":
        g_dev = [torch.zeros_like(upd, device=dev) for _ in range(world)]
        dist.all_gather(g_dev, upd.to(dev))
        gathered = [g.cpu() for g in g_dev]
    else:
        dist.all_gather(gathered, upd)
    if rank == 0:
        torch.manual_seed(5)
        net1 = AtariNet(num_actions=A, device=dev)
        opt1 = optim.RMSprop(net1.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
        q0 = net1.flat_params.clone()
        L1 = learner.FusedLearner(net1, flags, T, B)
        losses1 = L1.step(batch, None).clone()
        torch.cuda.synchronize()
        grads1 = net1.flat_grads.clone().cpu()
        L1.step(batch, opt1)
        torch.cuda.synchronize()
        upd1 = (net1.flat_params - q0).cpu()
        same = all(torch.equal(g, gathered[0]) for g in gathered)
        rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm())  # noqa: E731
        out_q.put((same, rel(grads, grads1), rel(upd, upd1), losses.cpu().tolist(), losses1.cpu().tolist()))
    dist.destroy_process_group()
