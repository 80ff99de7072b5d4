"""Seeded synthetic input generators shared by the tests, the bench and the oracle legs.

This module holds none of SPION's arithmetic (no convolution, pooling,
threshold, flood fill or attention).  It only draws inputs with the shapes
and structure of the paper's workloads (recipe in DESIGN.md §5):

* ``qkvdo``: Q, K, V, dO ~ N(0, 1) per (batch*head) slice, seeded per global
  slice index so any sharding over ranks regenerates identical slices.
* ``syn_mask``: the density-controlled block mask SYN(rho): forced diagonal,
  one vertical stripe, sub/super-diagonal band blocks, then uniform random
  blocks (the diagonal band and vertical stripes the paper observes).
* ``syn_scores``: a head-averaged attention-probability matrix A^s (rows sum
  to 1, values in [0, 1]) with a diagonal band and vertical stripes, the
  input of pattern generation.
"""
from __future__ import annotations

import math

import numpy as np
import torch


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def qkvdo(bh: int, L: int, d: int, seed: int = 1234, dtype=torch.bfloat16, device="cpu", start_bh: int = 0):
    """Return Q, K, V, dO of shape [bh, L, d] ~ N(0,1) rounded to ``dtype``.

    Slice b uses seeds ``seed + 4*(start_bh+b) + {0,1,2,3}`` on ``device``'s
    generator (CPU and CUDA streams differ; parity tests draw on CPU).
    """
    out = []
    for t in range(4):
        x = torch.empty((bh, L, d), dtype=torch.float32, device=device)
        for b in range(bh):
            g = _gen(seed + 4 * (start_bh + b) + t, device)
            x[b].normal_(0.0, 1.0, generator=g)
        out.append(x.to(dtype))
    return tuple(out)


def syn_mask(n: int, density: float = 0.10, seed: int = 7) -> np.ndarray:
    """SYN(rho): exactly max(n, round(rho*n*n)) blocks as uint8 [n][n]."""
    rng = np.random.default_rng(seed)
    target = max(n, int(round(density * n * n)))
    target = min(target, n * n)
    m = np.zeros((n, n), np.uint8)
    for k in range(n):
        m[k, k] = 1
    count = n

    def add(i, j):
        nonlocal count
        if count < target and not m[i, j]:
            m[i, j] = 1
            count += 1

    stripe = int(rng.integers(0, n))
    for i in range(n):
        add(i, stripe)
    band = [(i, i + 1) for i in range(n - 1)] + [(i + 1, i) for i in range(n - 1)]
    for k in rng.permutation(len(band)):
        add(*band[k])
    cells = [(i, j) for i in range(n) for j in range(n)]
    for k in rng.permutation(len(cells)):
        if count >= target:
            break
        add(*cells[k])
    return m


def syn_scores(L: int, B: int, heads: int = 4, seed: int = 11, n_stripes: int = 2, device="cpu") -> torch.Tensor:
    """Head-mean of row-softmax(4*exp(-((i-j)/(B/2))^2/2) + 3*[j in stripes] + N(0,1)), fp32 [L][L]."""
    g = _gen(seed, "cpu")
    stripes = torch.randint(0, L, (n_stripes,), generator=g)
    i = torch.arange(L, dtype=torch.float32, device=device)
    diff = (i[:, None] - i[None, :]) / (B / 2.0)
    base = 4.0 * torch.exp(-0.5 * diff * diff)
    stripe_col = torch.zeros(L, dtype=torch.float32, device=device)
    stripe_col[stripes.to(device)] = 3.0
    base = base + stripe_col[None, :]
    acc = torch.zeros((L, L), dtype=torch.float32, device=device)
    for h in range(heads):
        gh = _gen(seed * 1000003 + h, device)
        noise = torch.empty((L, L), dtype=torch.float32, device=device).normal_(0.0, 1.0, generator=gh)
        acc += torch.softmax(base + noise, dim=-1)
    acc /= heads
    return acc.clamp_(0.0, 1.0)


def lra_scores(L: int, B: int, seed: int = 1, device="cpu") -> torch.Tensor:
    """The benchmark's score matrix: ``syn_scores`` with 4 heads and n/8 stripe columns
    (n = L/B, at least 2), so the flood fill at alpha = 75 lands near the north star's
    ~10 % block density at every LRA shape."""
    return syn_scores(L, B, heads=4, seed=seed, n_stripes=max(2, (L // B) // 8), device=device)


def block_density(mask: np.ndarray) -> float:
    return float(np.asarray(mask).astype(bool).mean())

