"""Pins for the GQA head reduction and head policy of the oracle that a wrong reduction
cannot pass: closed-form per-key masses of one-hot / evenly split attention heads.

Construction (no formula of the oracle is retyped): d = 8 with RoPE base 1e300, so the rotate-half
pairs i = 1, 2, 3 (coordinates (1,5), (2,6), (3,7)) rotate by pos * 1e300^(-i/4) <= 1e-74 rad --
i.e. not at all in float64 -- and coordinate pair 0 is kept zero.  Four sink keys are unit vectors
e1, e2, e3 and 0; the chunk keys are 0.  A query 1000 * (sum of a subset of {e1, e2, e3}) puts
logit 1000/sqrt(8) ~ 354 on each key of the subset and <= 0 on every other visible key, so its
softmax row is uniform over the subset up to exp(-354) ~ 1e-154.  Every row of the chunk is the
same, so a head's per-key mass (Alg. 3) is f_j * sum_r C_EMA[r] = f_j * (1 - gamma^m) with
f_j the uniform fraction -- exact values to compare the reductions against:
    head A = e1        f = (1,   0,   0  )
    head B = e1 + e2   f = (1/2, 1/2, 0  )
    head C = e1+e2+e3  f = (1/3, 1/3, 1/3)
    head D = e2        f = (0,   1,   0  )
"""

import numpy as np
import pytest

from oracle.attention import reduce_heads
from oracle.model import CascadeOracle, OracleConfig

F = {"A": (1.0, 0.0, 0.0), "B": (0.5, 0.5, 0.0), "C": (1 / 3, 1 / 3, 1 / 3), "D": (0.0, 1.0, 0.0)}
Q = {"A": (1,), "B": (1, 2), "C": (1, 2, 3), "D": (2,)}
D_, GAMMA, M = 8, 0.9, 6


def _run(heads, num_kv_heads, how, policy="independent"):
    """Sinks hold e1, e2, e3, 0 (chunk 1, m = 4); chunk 2 (m = M) asks the queries.  Returns the
    chunk-2 scores of the four sink keys [B=1, Hkv, 4] (slots 0..3)."""
    Hq = len(heads)
    orc = CascadeOracle(OracleConfig(num_layers=1, batch=1, num_q_heads=Hq, num_kv_heads=num_kv_heads,
                                     head_dim=D_, sink_size=4, cache_size=8, num_cascades=2, gamma=GAMMA,
                                     rope_theta=1e300, head_reduce=how, head_policy=policy))
    k1 = np.zeros((1, 4, num_kv_heads, D_))
    for j in range(3):
        k1[0, j, :, 1 + j] = 1.0
    orc.prefill_stride(0, np.zeros((1, 4, Hq, D_)), k1, np.ones((1, 4, num_kv_heads, D_)))
    q = np.zeros((1, M, Hq, D_))
    for h, name in enumerate(heads):
        for c in Q[name]:
            q[0, :, h, c] = 1000.0
    k2 = np.zeros((1, M, num_kv_heads, D_))
    _, s = orc.prefill_stride(0, q, k2, np.ones((1, M, num_kv_heads, D_)))
    return s[0, :, :4]


def _mass(vals):
    return np.array(list(vals) + [0.0]) * (1 - GAMMA ** M)


def test_per_head_masses_are_the_closed_forms():
    for name in "ABCD":
        s = _run([name], 1, "max")
        np.testing.assert_allclose(s[0], _mass(F[name]), rtol=1e-12, atol=1e-15)


def test_group_max_mean_median_closed_forms():
    """G = 4 (A, B, C, D): max (1, 1, 1/3), mean (11/24, 11/24, 1/12), median of an even group =
    mean of the middle two ((1/3 + 1/2)/2, same, 0); the group SUM (11/6, 11/6, 1/3) would fail
    the max pin.  G = 3 (A, B, C): median (1/2, 1/3, 0)."""
    exp4 = {"max": (1, 1, 1 / 3), "mean": (11 / 24, 11 / 24, 1 / 12), "median": (5 / 12, 5 / 12, 0)}
    for how, vals in exp4.items():
        s = _run(list("ABCD"), 1, how)
        np.testing.assert_allclose(s[0], _mass(vals), rtol=1e-12, atol=1e-15)
    assert not np.allclose(_run(list("ABCD"), 1, "max")[0], _mass((11 / 6, 11 / 6, 1 / 3)))
    s = _run(list("ABC"), 1, "median")
    np.testing.assert_allclose(s[0], _mass((0.5, 1 / 3, 0)), rtol=1e-12, atol=1e-15)


def test_homogeneous_policy_reduces_over_all_heads():
    """Hq = 4, Hkv = 2 (groups {A, B}, {C, D}).  Independent max: kv-head 0 (1, 1/2, 0), kv-head 1
    (1/3, 1, 1/3).  Homogeneous max (one decision per sequence): both kv-heads get the max
    over all four heads, (1, 1, 1/3); homogeneous mean: the mean over all four, (11/24, 11/24, 1/12)."""
    s = _run(list("ABCD"), 2, "max")
    np.testing.assert_allclose(s[0], _mass((1, 0.5, 0)), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(s[1], _mass((1 / 3, 1, 1 / 3)), rtol=1e-12, atol=1e-15)
    for how, vals in (("max", (1, 1, 1 / 3)), ("mean", (11 / 24, 11 / 24, 1 / 12))):
        s = _run(list("ABCD"), 2, how, "homogeneous")
        for g in range(2):
            np.testing.assert_allclose(s[g], _mass(vals), rtol=1e-12, atol=1e-15)


def test_reduce_heads_hand_values():
    s = np.array([[1.0, 0.5], [0.25, 0.5], [0.0, 1.0], [0.75, 0.0]])
    np.testing.assert_array_equal(reduce_heads(s, 4, "max"), [[1.0, 1.0]])
    np.testing.assert_allclose(reduce_heads(s, 4, "mean"), [[0.5, 0.5]])
    np.testing.assert_allclose(reduce_heads(s, 4, "median"), [[0.5, 0.5]])      # (0.25+0.75)/2, (0.5+0.5)/2
    np.testing.assert_allclose(reduce_heads(s[:3], 3, "median"), [[0.25, 0.5]])
    np.testing.assert_allclose(reduce_heads(s[:3], 3, "mean"), [[1.25 / 3, 2 / 3]])


def test_homogeneous_median_score_injection_is_refused():
    """Homogeneous + median needs every q-head's mass; injected scores are per kv-head, so the
    oracle refuses instead of reducing the wrong quantity."""
    orc = CascadeOracle(OracleConfig(num_layers=1, batch=1, num_q_heads=4, num_kv_heads=2, head_dim=D_,
                                     sink_size=1, cache_size=4, num_cascades=2, head_reduce="median",
                                     head_policy="homogeneous"))
    with pytest.raises(ValueError):
        orc.update_with_scores(0, np.zeros((1, 1, 2, D_)), np.zeros((1, 1, 2, D_)), np.zeros((1, 2, 6)))
