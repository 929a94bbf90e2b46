"""Pins for the oracle's one-pass estimator of Alg. 3 (oracle.attention.key_mass_onepass):
a hand trace of the normaliser l_i + l_i rho / gamma over four inner steps, and the two cases
where the estimate is exact (one inner step; equal per-step sums)."""

import numpy as np
import pytest

from oracle.attention import key_mass, key_mass_onepass, chunk_attention
from oracle.model import CascadeOracle, OracleConfig


def test_hand_trace_four_inner_steps():
    """One query row, three single-key cache tiles with logits 0, ln 2, ln 3 and the row's own
    key at logit -1000 (gamma = 0, so C_EMA = 1 for the single row).  Step j (1-based) sees the
    running sum l_j = 1, 3, 6, 6 and divides by l_j (1 + (4 - j) / j):
        key 0: 1 / (1 * 4)       = 1/4
        key 1: 2 / (3 * (1 + 1)) = 1/3
        key 2: 3 / (6 * (4/3))   = 3/8
        key 3: e^-1000 / 6       = 0
    whereas the exact masses are 1/6, 1/3, 1/2, 0."""
    q = np.array([[1.0]])
    k = np.array([[0.0], [np.log(2.0)], [np.log(3.0)], [-1000.0]])
    s = key_mass_onepass(q, k, 3, 1.0, 0.0, [[0], [1], [2]], q_tile=1)
    np.testing.assert_allclose(s, [0.25, 1 / 3, 0.375, 0.0], rtol=1e-14, atol=1e-300)
    _, P = chunk_attention(q, k, np.zeros((4, 1)), 3, 1.0)
    np.testing.assert_allclose(key_mass(P, 0.0), [1 / 6, 1 / 3, 0.5, 0.0], rtol=1e-14, atol=1e-300)


def test_single_inner_step_is_exact():
    """With every key in one tile (no cache, one chunk tile) the normaliser at the only step is
    the final row sum: the estimate equals the exact mass."""
    rng = np.random.default_rng(3)
    m, d = 9, 8
    q, k = rng.standard_normal((m, d)), rng.standard_normal((m, d))
    s = key_mass_onepass(q, k, 0, 0.3, 0.9, [], q_tile=16)
    _, P = chunk_attention(q, k, np.zeros((m, d)), 0, 0.3)
    np.testing.assert_allclose(s, key_mass(P, 0.9), rtol=1e-13)


def test_equal_step_sums_are_exact():
    """Equal logits and single-key tiles: each inner step adds the same amount to l, so
    l_j (1 + rho/gamma) = l_j n / j = the final sum at every step and the estimate is exact."""
    q = np.zeros((1, 4))
    k = np.zeros((5, 4))
    s = key_mass_onepass(q, k, 4, 1.0, 0.5, [[0], [1], [2], [3]], q_tile=1)
    np.testing.assert_allclose(s, np.full(5, 0.5 / 5), rtol=1e-14)


def test_oracle_onepass_mode_uses_the_flat_slot_tiles():
    """In the model, onepass mode differs from exact mode only through the per-key mass: the
    outputs of a chunk are identical; decode steps use the exact mass in both modes."""
    rng = np.random.default_rng(5)
    base = dict(num_layers=1, batch=1, num_q_heads=2, num_kv_heads=1, head_dim=8, sink_size=2,
                cache_size=12, num_cascades=3, gamma=0.95)
    ex = CascadeOracle(OracleConfig(**base))
    op = CascadeOracle(OracleConfig(score_mode="onepass", tile=4, **base))
    for _ in range(5):
        q, k, v = rng.standard_normal((1, 6, 2, 8)), rng.standard_normal((1, 6, 1, 8)), rng.standard_normal((1, 6, 1, 8))
        o1, s1 = ex.prefill_stride(0, q, k, v)
        o2, s2 = op.prefill_stride(0, q, k, v)
        np.testing.assert_array_equal(o1, o2)
        assert s2.sum() > 0 and np.all(s2 >= 0)
    # decode steps use the exact mass in both modes
    ex, op = CascadeOracle(OracleConfig(**base)), CascadeOracle(OracleConfig(score_mode="onepass", tile=4, **base))
    for _ in range(20):
        q, k, v = (rng.standard_normal((1, 2, 8)), rng.standard_normal((1, 1, 8)), rng.standard_normal((1, 1, 8)))
        np.testing.assert_array_equal(ex.decode(0, q, k, v)[1], op.decode(0, q, k, v)[1])
