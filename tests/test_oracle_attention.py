"""Pins for the attention half of the oracle (Eq. 5, Alg. 5/6).

P8/P9: library routine (torch scaled_dot_product_attention in fp64, autograd
for the backward); P10: PAPER/MASKED closed form; P11: implicit-zero identity;
P12 and the SDDMM example: worked examples (tests/golden); P13: central finite
differences; P14: locality.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from synth import syn_mask


def _rand(L, d, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((L, d)) for _ in range(4)]


def _sdpa(Q, K, V, mask_dense, scale):
    q, k, v = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (Q, K, V))
    attn_mask = None if mask_dense is None else torch.tensor(mask_dense.astype(bool))
    o = torch.nn.functional.scaled_dot_product_attention(q[None, None], k[None, None], v[None, None],
                                                         attn_mask=attn_mask, scale=scale)[0, 0]
    return q, k, v, o


def _dense(fl, B):
    return np.kron(fl, np.ones((B, B), np.uint8))


@pytest.mark.parametrize("L,d,B", [(16, 4, 4), (32, 8, 8), (64, 16, 8)])
def test_p8_all_ones_mask_is_dense_attention(L, d, B):
    Q, K, V, dO = _rand(L, d, L + d)
    fl = np.ones((L // B, L // B), np.uint8)
    scale = 1.0 / math.sqrt(d)
    q, k, v, o = _sdpa(Q, K, V, None, scale)
    o.backward(torch.tensor(dO))
    for mode in ("paper", "masked"):
        O, lse = oracle.attn_fwd(Q, K, V, fl, B, scale, mode)
        assert np.abs(O - o.detach().numpy()).max() < 1e-12
        dQ, dK, dV = oracle.attn_bwd(Q, K, V, dO, fl, B, scale, mode)
        assert np.abs(dQ - q.grad.numpy()).max() < 1e-12
        assert np.abs(dK - k.grad.numpy()).max() < 1e-12
        assert np.abs(dV - v.grad.numpy()).max() < 1e-12


@pytest.mark.parametrize("L,d,B,density", [(32, 8, 4, 0.3), (64, 16, 8, 0.2), (48, 4, 16, 0.5)])
def test_p9_masked_mode_is_sdpa_with_boolean_mask(L, d, B, density):
    Q, K, V, dO = _rand(L, d, 7 * L + B)
    fl = syn_mask(L // B, density, seed=L)
    scale = 0.37
    q, k, v, o = _sdpa(Q, K, V, _dense(fl, B), scale)
    o.backward(torch.tensor(dO))
    O, lse = oracle.attn_fwd(Q, K, V, fl, B, scale, "masked")
    assert np.abs(O - o.detach().numpy()).max() < 1e-12
    dQ, dK, dV = oracle.attn_bwd(Q, K, V, dO, fl, B, scale, "masked")
    assert np.abs(dQ - q.grad.numpy()).max() < 1e-12
    assert np.abs(dK - k.grad.numpy()).max() < 1e-12
    assert np.abs(dV - v.grad.numpy()).max() < 1e-12


def test_p10_paper_vs_masked_closed_form():
    """lse_P = logaddexp(lse_M, ln(L - cnt)); O_P = O_M * exp(lse_M - lse_P)."""
    L, d, B = 64, 16, 8
    Q, K, V, _ = _rand(L, d, 3)
    Q *= 3.0  # wide logits
    fl = syn_mask(L // B, 0.25, seed=2)
    scale = 1.0 / math.sqrt(d)
    OP, lseP = oracle.attn_fwd(Q, K, V, fl, B, scale, "paper")
    OM, lseM = oracle.attn_fwd(Q, K, V, fl, B, scale, "masked")
    cnt = np.repeat(fl.sum(1) * B, B)
    assert np.abs(lseP - np.logaddexp(lseM, np.log(L - cnt))).max() < 1e-12
    assert np.abs(OP - OM * np.exp(lseM - lseP)[:, None]).max() < 1e-12


def test_p11_implicit_zero_identity():
    L, d, B = 32, 8, 4
    Q, K, V, _ = _rand(L, d, 5)
    fl = syn_mask(L // B, 0.3, seed=1)
    scale = 0.5
    _, lseP, PP = oracle.attn_fwd(Q, K, V, fl, B, scale, "paper", want_P=True)
    _, lseM, PM = oracle.attn_fwd(Q, K, V, fl, B, scale, "masked", want_P=True)
    cnt = np.repeat(fl.sum(1) * B, B)
    assert np.abs(PP.sum(1) + (L - cnt) * np.exp(-lseP) - 1.0).max() < 1e-12
    assert np.abs(PM.sum(1) - 1.0).max() < 1e-12
    # probabilities vanish off the mask (Eq. 5 / SpMM over stored entries only)
    assert (PP[_dense(fl, B) == 0] == 0).all()


def test_p12_sparse_softmax_worked_example(golden_dir):
    with open(os.path.join(golden_dir, "sparse_softmax_spec.json")) as f:
        g = json.load(f)
    L, B, d = g["L"], 2, 3
    Q = np.zeros((L, d))  # all stored logits 0
    rng = np.random.default_rng(0)
    K, V = rng.standard_normal((L, d)), rng.standard_normal((L, d))
    fl = np.array([[1, 0], [0, 1]], np.uint8)  # row 0 stores exactly 2 entries
    for mode in ("paper", "masked"):
        _, _, P = oracle.attn_fwd(Q, K, V, fl, B, 1.0, mode, want_P=True)
        assert np.allclose(P[0, :2], g[mode], atol=0, rtol=1e-15)


def test_sddmm_worked_example(golden_dir):
    with open(os.path.join(golden_dir, "sddmm_spec.json")) as f:
        g = json.load(f)
    Q, K = np.array(g["Q"], float), np.array(g["K"], float)
    V = np.array([[1.0, 1.0], [3.0, 4.0]])
    fl = np.array(g["pattern"], np.uint8)
    O, lse = oracle.attn_fwd(Q, K, V, fl, 1, 1.0, "masked")
    assert list(lse) == g["sddmm"]  # one stored entry per row: lse = stored logit
    assert (O == V).all()


def test_empty_rows_conventions():
    L, d, B = 16, 4, 4
    Q, K, V, dO = _rand(L, d, 11)
    fl = np.eye(4, dtype=np.uint8)
    fl[2, 2] = 0  # block-row 2 empty (only possible for user masks)
    for mode, want in (("paper", math.log(L)), ("masked", -math.inf)):
        O, lse = oracle.attn_fwd(Q, K, V, fl, B, 0.5, mode)
        assert (O[8:12] == 0).all()
        assert (lse[8:12] == want).all()
        dQ, dK, dV = oracle.attn_bwd(Q, K, V, dO, fl, B, 0.5, mode)
        assert (dQ[8:12] == 0).all() and (dK[8:12] == 0).all() and (dV[8:12] == 0).all()


@pytest.mark.parametrize("mode", ["paper", "masked"])
def test_p13_finite_differences(mode):
    L, d, B = 16, 4, 4
    rng = np.random.default_rng(42 if mode == "paper" else 43)
    Q, K, V, dO = (rng.standard_normal((L, d)) for _ in range(4))
    fl = syn_mask(L // B, 0.4, seed=3)
    scale = 0.6
    dQ, dK, dV = oracle.attn_bwd(Q, K, V, dO, fl, B, scale, mode)

    def loss(Qx, Kx, Vx):
        O, _ = oracle.attn_fwd(Qx, Kx, Vx, fl, B, scale, mode)
        return float((O * dO).sum())

    eps = 1e-6
    for X, G, which in ((Q, dQ, 0), (K, dK, 1), (V, dV, 2)):
        num = np.zeros_like(X)
        for idx in np.ndindex(*X.shape):
            args_p = [Q.copy(), K.copy(), V.copy()]
            args_m = [Q.copy(), K.copy(), V.copy()]
            args_p[which][idx] += eps
            args_m[which][idx] -= eps
            num[idx] = (loss(*args_p) - loss(*args_m)) / (2 * eps)
        rel = np.abs(num - G).max() / max(1e-12, np.abs(G).max())
        assert rel < 1e-6, (which, rel)


def test_p14_locality_block_diagonal():
    L, d, B = 32, 8, 8
    Q, K, V, _ = _rand(L, d, 13)
    fl = np.eye(L // B, dtype=np.uint8)
    O1, _ = oracle.attn_fwd(Q, K, V, fl, B, 0.4, "paper")
    V2 = V.copy()
    V2[8:16] += 100.0  # outside block-row 0's stored blocks
    O2, _ = oracle.attn_fwd(Q, K, V2, fl, B, 0.4, "paper")
    assert (O1[:8] == O2[:8]).all()
    assert not (O1[8:16] == O2[8:16]).all()


# ------------------------------------------------------ NEXT-1: dense-phase score capture
def test_score_mean_matches_torch_softmax():
    """A^s = mean over (batch, head) of softmax(scale Q K^T): against torch.softmax in fp64 (library
    routine), rows sum to 1, and the sum of squares against numpy."""
    rng = np.random.default_rng(3)
    bh, L, d = 5, 48, 8
    Q, K = rng.standard_normal((bh, L, d)), rng.standard_normal((bh, L, d))
    scale = 1 / math.sqrt(d)
    A, ss = oracle.score_mean(Q, K, scale)
    ref = torch.softmax(torch.from_numpy(Q) @ torch.from_numpy(K).transpose(1, 2) * scale, dim=-1).mean(0).numpy()
    assert np.abs(A - ref).max() < 1e-14
    assert np.abs(A.sum(1) - 1).max() < 1e-12
    assert abs(ss - float((ref ** 2).sum())) < 1e-12


def test_transition_eq2_worked_numbers():
    """Eq. 2 / Alg. 2 by hand: norms 3, 2.5, 2.2 -> distances 0.5, 0.3, |0.5 - 0.3| = 0.2."""
    ok, d1, d2 = oracle.transition(9.0, 6.25, 4.84, 0.25)
    assert ok and abs(d1 - 0.5) < 1e-12 and abs(d2 - 0.3) < 1e-12
    ok, _, _ = oracle.transition(9.0, 6.25, 4.84, 0.15)
    assert not ok
