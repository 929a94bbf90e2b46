"""Pins for oracle/stack.py (Alg. 1's layer loop over coupled synthetic attention layers,
PAPER.md:106-119) against an independent dense computation: below the
first drop no token has left the cascade (S <= alpha + 2c is always safe), so
every layer's strided attention equals full causal attention at absolute positions, and the
stack equals a dense causal multi-layer attention stack built from torch SDPA (float64) and a
complex-number RoPE -- code that shares nothing with the oracle."""

import numpy as np
import pytest
import torch

from oracle.stack import StackOracle, stack_config


def _rope_complex(x, pos, theta):
    d = x.shape[-1]
    z = x[..., : d // 2] + 1j * x[..., d // 2:]
    freqs = np.array([theta ** (-2.0 * i / d) for i in range(d // 2)])
    z = z * np.exp(1j * np.multiply.outer(pos, freqs))
    return np.concatenate([z.real, z.imag], axis=-1)


def _dense_stack(x, wq, wk, wv, wo, Hq, Hk, d, theta):
    """Full causal attention stack: x <- x + SDPA(rope(x Wq), rope(x Wk), x Wv) Wo, per layer."""
    B, S, D = x.shape
    G = Hq // Hk
    pos = np.arange(S)
    for l in range(len(wq)):
        q = (x @ wq[l]).reshape(B, S, Hq, d)
        k = (x @ wk[l]).reshape(B, S, Hk, d)
        v = (x @ wv[l]).reshape(B, S, Hk, d)
        qr = np.stack([_rope_complex(q[:, :, h], pos, theta) for h in range(Hq)], axis=2)
        kr = np.stack([_rope_complex(k[:, :, g], pos, theta) for g in range(Hk)], axis=2)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).double().permute(0, 2, 1, 3)
        kt = t(kr).repeat_interleave(G, dim=1)
        vt = t(v).repeat_interleave(G, dim=1)
        O = torch.nn.functional.scaled_dot_product_attention(t(qr), kt, vt, is_causal=True)
        O = O.permute(0, 2, 1, 3).numpy().reshape(B, S, Hq * d)
        x = x + O @ wo[l]
    return x


def _weights(rng, L, D, Hq, Hk, d, wo_scale=1.0):
    s = 1.0 / np.sqrt(D)
    wq = [rng.standard_normal((D, Hq * d)) * s for _ in range(L)]
    wk = [rng.standard_normal((D, Hk * d)) * s for _ in range(L)]
    wv = [rng.standard_normal((D, Hk * d)) * s for _ in range(L)]
    wo = [rng.standard_normal((Hq * d, D)) * s * wo_scale for _ in range(L)]
    return wq, wk, wv, wo


@pytest.mark.parametrize("stride", [1, 7, 24])
def test_stack_below_first_drop_equals_dense_causal_stack(stride):
    """alpha = 4, N = 3, c = 8: the first drop is at t >= alpha + 2c = 20 (App. B.3); 20 tokens of
    a 3-layer GQA stack (Hq 4, Hkv 2, d 8, D 32) at strides 1, 7 and one 20-token chunk."""
    L, B, Hq, Hk, d, D, S, theta = 3, 2, 4, 2, 8, 32, 20, 10000.0
    rng = np.random.default_rng(11)
    wq, wk, wv, wo = _weights(rng, L, D, Hq, Hk, d)
    x = rng.standard_normal((B, S, D))
    cfg = stack_config(L, B, Hq, Hk, d, 4, 24, 3, rope_theta=theta, gamma=0.9)
    orc = StackOracle(cfg, wq, wk, wv, wo)
    outs = []
    for a in range(0, S, stride):
        outs.append(orc.prefill_stride(x[:, a:a + stride]))
    got = np.concatenate(outs, axis=1)
    ref = _dense_stack(x, wq, wk, wv, wo, Hq, Hk, d, theta)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-11)
    for l in range(L):                       # nothing dropped yet: every token is resident
        org = orc.state(l)["origin"]
        assert sorted(org[org >= 0].tolist()) == sorted(list(range(S)) * (B * Hk))


def test_stack_layers_are_coupled_through_the_residual_stream():
    """Layer l+1's keys are projections of layer l's output (Alg. 1 runs the layers of a chunk in
    order): with W_o = 0 every layer sees the chunk input itself (x unchanged, all layers' cascades
    hold keys x W_k^l); changing layer 0's W_o changes layer 1's cached keys but not layer 0's."""
    L, B, Hq, Hk, d, D, m = 2, 1, 2, 1, 8, 16, 6
    rng = np.random.default_rng(5)
    wq, wk, wv, wo = _weights(rng, L, D, Hq, Hk, d)
    x = rng.standard_normal((B, 3 * m, D))
    cfg = stack_config(L, B, Hq, Hk, d, 2, 8, 2, rope_theta=10000.0)
    zero = StackOracle(cfg, wq, wk, wv, [np.zeros_like(w) for w in wo])
    for a in range(0, 3 * m, m):
        np.testing.assert_array_equal(zero.prefill_stride(x[:, a:a + m]), x[:, a:a + m])
    for l in range(L):
        st = zero.state(l)
        for sl in np.flatnonzero(st["origin"][0, 0] >= 0):
            t = st["origin"][0, 0, sl]
            np.testing.assert_allclose(st["k"][0, 0, sl], x[0, t] @ wk[l], rtol=0, atol=1e-12)
    a = StackOracle(cfg, wq, wk, wv, wo)
    wo2 = [wo[0] * 2.0, wo[1]]
    b = StackOracle(cfg, wq, wk, wv, wo2)
    for c in range(0, 3 * m, m):
        a.prefill_stride(x[:, c:c + m])
        b.prefill_stride(x[:, c:c + m])
    np.testing.assert_array_equal(a.state(0)["k"], b.state(0)["k"])
    assert np.abs(a.state(1)["k"] - b.state(1)["k"]).max() > 1e-3


def test_stack_bf16_io_rounds_every_intermediate():
    """round_bf16_io: q, k, v, O and the residual stream are bf16 values (torch's RNE rounding)."""
    L, B, Hq, Hk, d, D, m = 2, 1, 4, 2, 8, 32, 5
    rng = np.random.default_rng(9)
    wq, wk, wv, wo = _weights(rng, L, D, Hq, Hk, d)
    cfg = stack_config(L, B, Hq, Hk, d, 2, 8, 2, rope_theta=10000.0)
    orc = StackOracle(cfg, wq, wk, wv, wo, round_bf16_io=True)
    x = rng.standard_normal((B, m, D))
    y = orc.prefill_stride(x)
    is_bf16 = lambda a: np.array_equal(torch.from_numpy(a).to(torch.bfloat16).double().numpy(), a)
    assert is_bf16(y)
    for tr in orc.trace:
        for key in ("x", "q", "k", "v", "O"):
            assert is_bf16(tr[key]), key
    xb = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(orc.trace[0]["x"], xb)
    np.testing.assert_array_equal(
        orc.trace[0]["q"].reshape(B, m, -1), torch.from_numpy(xb @ wq[0]).to(torch.bfloat16).double().numpy())
