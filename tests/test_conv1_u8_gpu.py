"""conv1 with its A operand built on chip from the u8 frames (bulk-copied frame lines ->
converter warps -> 128B-swizzled bf16 window, GEMM engine AU8 mode) must be bit-identical to
the bf16 space-to-depth grid path: the same bf16 operands reach the same MMAs."""
import pytest
import torch

from paper_1910_03552_b200 import _native as N

pytestmark = pytest.mark.gpu


def _run(net, frames, reward, la, mode, **kw):
    prev = N.lib().bp_atari_set_conv1_u8(mode)
    try:
        lg, bl = net._forward_kernels(frames, reward, la, repack=True, **kw)
        return lg.clone(), bl.clone()
    finally:
        N.lib().bp_atari_set_conv1_u8(prev)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("n", [1, 7, 64, 300])
def test_conv1_u8_forward_bit_identical(n, mode):
    from paper_1910_03552_b200.atari_net import AtariNet

    torch.manual_seed(n)
    net = AtariNet(num_actions=6)
    frames = torch.randint(0, 256, (n, 4, 84, 84), dtype=torch.uint8, device="cuda")
    reward = torch.rand(n, device="cuda")
    la = torch.randint(0, 6, (n,), device="cuda")
    a = _run(net, frames, reward, la, 0)
    b = _run(net, frames, reward, la, mode)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("mode", [1, 2])
def test_conv1_u8_plane_store_bit_identical(mode):
    from paper_1910_03552_b200 import rollout
    from paper_1910_03552_b200.atari_net import AtariNet

    T, B = 9, 5
    torch.manual_seed(3)
    net = AtariNet(num_actions=6)
    done = torch.rand(T + 1, B) < 0.2
    planes = torch.randint(0, 256, (T + 4, B, 84, 84), dtype=torch.uint8, device="cuda")
    idx = rollout.frame_stack_index(done).cuda()
    frames = rollout.stack_frames(planes, idx).reshape(-1, 4, 84, 84)
    n = frames.shape[0]
    reward = torch.rand(n, device="cuda")
    la = torch.randint(0, 6, (n,), device="cuda")
    a = _run(net, frames, reward, la, 0)
    b = _run(net, planes, reward, la, mode, plane_index=idx.reshape(n, 4))
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("mode", [1, 2])
def test_conv1_u8_backward_bit_identical(mode):
    """The converter's X0 side output feeds the conv1 weight gradient: whole-network
    gradients must equal the space-to-depth path bit for bit."""
    from paper_1910_03552_b200.atari_net import AtariNet

    n = 200
    torch.manual_seed(11)
    net = AtariNet(num_actions=6)
    frames = torch.randint(0, 256, (n, 4, 84, 84), dtype=torch.uint8, device="cuda")
    reward = torch.rand(n, device="cuda")
    la = torch.randint(0, 6, (n,), device="cuda")
    dl = torch.randn(n, 6, device="cuda")
    db = torch.randn(n, device="cuda")
    grads = []
    for m in (0, mode):
        prev = N.lib().bp_atari_set_conv1_u8(m)
        try:
            net._forward_kernels(frames, reward, la, repack=True)
            g = torch.empty_like(net.flat_params)
            net._backward_kernels(dl, db, reward, la, g)
            grads.append(g)
        finally:
            N.lib().bp_atari_set_conv1_u8(prev)
    assert torch.equal(grads[0], grads[1])
