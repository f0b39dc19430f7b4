"""flatten_params (paper_2604_07808_b200.torch_blocks, CPU): a block's
parameters become views of ONE flat buffer (the library's layer unit,
include/grass.h) and autograd accumulates their gradients into ONE flat
gradient buffer, in parameter order."""
import torch

from paper_2604_07808_b200.torch_blocks import flatten_params


def test_flatten_params_views_and_gradients():
    torch.manual_seed(0)
    block = torch.nn.Sequential(torch.nn.Linear(5, 7), torch.nn.GELU(), torch.nn.Linear(7, 3))
    before = [p.detach().clone() for p in block.parameters()]
    flat, gflat = flatten_params(block.parameters())
    assert flat.numel() == sum(p.numel() for p in before) == gflat.numel()
    off = 0
    for p, b in zip(block.parameters(), before):
        assert torch.equal(p.detach(), b)                               # values kept
        assert p.data_ptr() == flat[off:].data_ptr()                    # a view of the flat buffer
        assert p.grad.data_ptr() == gflat[off:].data_ptr()
        off += p.numel()
    x = torch.randn(4, 5)
    block(x).square().sum().backward()
    ref = torch.nn.Sequential(torch.nn.Linear(5, 7), torch.nn.GELU(), torch.nn.Linear(7, 3))
    with torch.no_grad():
        for q, b in zip(ref.parameters(), before):
            q.copy_(b)
    ref(x).square().sum().backward()
    assert torch.allclose(gflat, torch.cat([q.grad.reshape(-1) for q in ref.parameters()]))
    flat.add_(1.0)                                                      # an update of the flat buffer
    assert torch.equal(next(block.parameters()).detach(), before[0] + 1.0)
