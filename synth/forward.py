"""Synthetic Llama forward used ONLY as a load generator for the prefetch-overlap
measurement (Alg. 1 l.408-412: each module's forward runs right after
its sync).  Not part of the method.  Per unit on the compute stream:

* embed : x = W_emb[ids]                                 (gather)
* layer : bf16 GEMMs q,k,v,o (h x h), gate, up (I x h), down (h x I) on x, residual adds
          (the attention core is omitted; SURVEY 8d sizes the forward by these GEMMs)
* head  : logits = x W_lm^T                              (T x V)

The weights are views into the unit's synced `local` buffer when the mesh has M == 1 (so the
forward really reads what the sync wrote); for M > 1 (sharded units, the FSDP all-gather is
out of scope) they are views into a per-rank full-size stand-in buffer.
"""
from __future__ import annotations

import torch

from . import LLAMA, VOCAB, Unit


class SyntheticForward:
    def __init__(self, model: str, units: list[Unit], tokens: int, device, dtype=torch.bfloat16, seed: int = 7):
        self.h, self.inter = LLAMA[model]
        self.units, self.tokens, self.device, self.dtype = units, tokens, device, dtype
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        self.ids = torch.randint(0, VOCAB, (tokens,), generator=g, device=device)
        self.x = torch.empty(tokens, self.h, dtype=dtype, device=device)
        self.standin = None

    def flops_per_round(self) -> float:
        h, i, T = self.h, self.inter, self.tokens
        layer = 2 * T * (4 * h * h + 3 * h * i)
        return 32 * layer + 2 * T * h * VOCAB

    def _weights(self, u: int, local: torch.Tensor) -> torch.Tensor:
        full = self.units[u].numel
        if local.numel() >= full:
            return local[:full]
        if self.standin is None or self.standin.numel() < full:
            self.standin = torch.randn(max(x.numel for x in self.units), device=self.device).mul_(0.02).to(self.dtype)
        return self.standin[:full]

    def unit(self, u: int, local: torch.Tensor) -> None:
        h, inter, T = self.h, self.inter, self.tokens
        w = self._weights(u, local)
        if self.dtype != w.dtype:
            w = w.to(self.dtype)
        if u == 0:  # embedding
            torch.index_select(w.view(VOCAB, h), 0, self.ids, out=self.x)
            return
        if u == len(self.units) - 1:  # final norm + lm head
            lm = w[h:].view(VOCAB, h)
            xn = self.x * w[:h]
            torch.matmul(xn, lm.t())
            return
        o = 0
        def take(rows, cols):
            nonlocal o
            m = w[o:o + rows * cols].view(rows, cols)
            o += rows * cols
            return m
        wq, wk, wv, wo = take(h, h), take(h, h), take(h, h), take(h, h)
        wg, wu, wd = take(inter, h), take(inter, h), take(h, inter)
        n1, n2 = w[o:o + h], w[o + h:o + 2 * h]
        x = self.x
        xn = x * n1
        q = xn @ wq.t()
        k = xn @ wk.t()
        v = xn @ wv.t()
        attn = v + 0.0 * (q[:, :1] + k[:, :1])  # attention core omitted; keep q, k live
        x = x + attn @ wo.t()
        xn = x * n2
        a = torch.nn.functional.silu(xn @ wg.t()) * (xn @ wu.t())
        self.x = x + a @ wd.t()
