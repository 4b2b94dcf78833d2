"""Switch/BERT-MoE encoder stack around MoELayer (BASELINE.json configs[4]).

The reference models one MoE layer and says to "compose layers externally"
(README.md:151-152).  This is that composition: a
pre-LN BERT block whose FFN is the pipelined expert-parallel MoELayer
(Switch Transformer style: top-1, capacity factor 1.25), attention and
LayerNorm from stock PyTorch (cuBLAS projections + the fused SDPA kernel;
library code, not part of the hot path).  Config 5: 12 blocks, d_model
1024, d_ffn 4096, 128 experts, sequence 1024.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn

from .layer import MoELayer


class MoEEncoderBlock(nn.Module):
    """x + Attn(LN(x)); x + MoE(LN(x))  (pre-LN; bf16 activations)."""

    def __init__(self, d_model: int, n_heads: int, d_ffn: int, num_experts: int, top_k: int = 1,
                 capacity_factor: float = 1.25, dtype=torch.bfloat16, device=None, layer_index: int = 0,
                 **moe_kw) -> None:
        super().__init__()
        if d_model % n_heads:
            raise ValueError("d_model must be divisible by n_heads")
        self.n_heads = n_heads
        fk = dict(dtype=dtype, device=device)
        self.ln1 = nn.LayerNorm(d_model, **fk)
        self.qkv = nn.Linear(d_model, 3 * d_model, **fk)
        self.proj = nn.Linear(d_model, d_model, **fk)
        self.ln2 = nn.LayerNorm(d_model, **fk)
        self.moe = MoELayer(d_model, d_ffn, num_experts, top_k=top_k, capacity_factor=capacity_factor,
                            dtype=dtype, device=device, seed=1000 * layer_index, **moe_kw)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        B, S, D = x.shape
        q, k, v = self.qkv(self.ln1(x)).view(B, S, 3, self.n_heads, D // self.n_heads).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(q, k, v)
        x = x + self.proj(a.transpose(1, 2).reshape(B, S, D))
        return x + self.moe(self.ln2(x).reshape(B * S, D)).view(B, S, D)


class MoEEncoder(nn.Module):
    """`layers` MoEEncoderBlocks (config 5: 12 x (1024, 16 heads, 4096, 128 experts top-1, cf 1.25))."""

    def __init__(self, layers: int = 12, d_model: int = 1024, n_heads: int = 16, d_ffn: int = 4096,
                 num_experts: int = 128, top_k: int = 1, capacity_factor: float = 1.25, dtype=torch.bfloat16,
                 device=None, **moe_kw) -> None:
        super().__init__()
        self.blocks = nn.ModuleList(
            MoEEncoderBlock(d_model, n_heads, d_ffn, num_experts, top_k, capacity_factor, dtype, device, i,
                            **moe_kw) for i in range(layers))
        self.ln_f = nn.LayerNorm(d_model, dtype=dtype, device=device)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        for blk in self.blocks:
            x = blk(x)
        return self.ln_f(x)

    def moe_layers(self) -> list[MoELayer]:
        return [b.moe for b in self.blocks]
