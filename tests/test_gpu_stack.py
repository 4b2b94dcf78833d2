"""The Switch/BERT-MoE stack (BASELINE configs[4] composition, stack.py):
gradients through attention + LayerNorm + MoELayer blocks agree with finite
differences of the loss (fp32 end to end, so the check is tight), and the
bf16 stack is deterministic run to run."""

import pytest
import torch

from paper_2506_22175_b200.stack import MoEEncoder

pytestmark = pytest.mark.gpu


def _ref_moe(x2, moe, idx, slot):
    """Differentiable torch restatement of one MoE layer (fp32) given its routing decisions."""
    logits = x2 @ moe.gate_weight.t()
    k = idx.shape[1]
    probs = torch.softmax(logits, dim=-1)
    chosen = torch.gather(logits, 1, idx.long())
    w = torch.gather(probs, 1, idx.long()) if k == 1 else torch.softmax(chosen, dim=-1)
    y = torch.zeros_like(x2)
    for j in range(k):
        for e in range(moe.num_experts):
            sel = ((idx[:, j] == e) & (slot[:, j] >= 0)).nonzero().flatten()
            if sel.numel():
                h = torch.relu(x2[sel] @ moe.w1[e].t()) @ moe.w2[e].t()
                y = y.index_add(0, sel, w[sel, j:j + 1] * h)
    return y


def _ref_forward(model, x, routes):
    for blk, (idx, slot) in zip(model.blocks, routes):
        B, S, D = x.shape
        q, k, v = blk.qkv(blk.ln1(x)).view(B, S, 3, blk.n_heads, D // blk.n_heads).permute(2, 0, 3, 1, 4)
        a = torch.nn.functional.scaled_dot_product_attention(q, k, v)
        x = x + blk.proj(a.transpose(1, 2).reshape(B, S, D))
        x = x + _ref_moe(blk.ln2(x).reshape(B * S, D), blk.moe, idx, slot).view(B, S, D)
    return model.ln_f(x)


@pytest.mark.parametrize("n,k", [(1, 1), (2, 1), (2, 2)])
def test_stack_gradients_match_torch_reference_fp32(cuda, n, k):
    """Every parameter gradient of the composed stack (attention + LN + our MoELayer) equals
    autograd through a plain-PyTorch fp32 restatement fed the same routing decisions."""
    torch.manual_seed(0)
    model = MoEEncoder(layers=2, d_model=128, n_heads=4, d_ffn=256, num_experts=8, top_k=k, capacity_factor=1.25,
                       dtype=torch.float32, device=cuda, pipeline=n)
    x = torch.randn(2, 64, 128, device=cuda, requires_grad=True)
    w = torch.randn(2, 64, 128, device=cuda)
    params = [x] + list(model.parameters())
    y = model(x)
    routes = [(b.moe.last_arena.idx.clone(), b.moe.last_arena.slot.clone()) for b in model.blocks]
    got = torch.autograd.grad((y * w).sum(), params)
    y_ref = _ref_forward(model, x, routes)
    want = torch.autograd.grad((y_ref * w).sum(), params)
    torch.testing.assert_close(y, y_ref, rtol=1e-4, atol=1e-4)
    for g_, w_ in zip(got, want):
        torch.testing.assert_close(g_, w_, rtol=1e-3, atol=1e-4 * max(w_.abs().max().item(), 1e-6))


def test_stack_bf16_deterministic(cuda):
    model = MoEEncoder(layers=2, d_model=256, n_heads=4, d_ffn=512, num_experts=16, device=cuda, pipeline=2)
    g = torch.Generator(device=cuda).manual_seed(1)
    x = torch.randn(2, 128, 256, device=cuda, generator=g, dtype=torch.bfloat16)
    outs = []
    for _ in range(2):
        xi = x.clone().requires_grad_(True)
        y = model(xi)
        y.float().square().sum().backward()
        outs.append((y.detach().clone(), xi.grad.clone(), model.blocks[0].moe.w1.grad.clone()))
        for p in model.parameters():
            p.grad = None
    for a, b in zip(*outs):
        assert torch.isfinite(a.float()).all()
        assert torch.equal(a, b)
