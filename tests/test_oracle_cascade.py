"""Pins for oracle/cascade.py (Alg. 2) against what the paper and brute force fix."""

import os
import random

import numpy as np
import pytest

from oracle.accounting import sparsity, stride_chunks, token_span
from oracle.cascade import CascadeHead, Ring, Token, reindex_positions
from oracle.model import CascadeOracle, OracleConfig
from oracle.naive import NaiveCascade

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load_toy_trace():
    rows = []
    with open(os.path.join(GOLDEN, "toy_trace_alpha1_N2_c2.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            t, mu, l1, x1, l2, x2, order = [c.strip() for c in line.split("|")]
            rows.append(dict(t=int(t), mu=float(mu),
                             l1=[None if s == "-" else int(s) for s in l1.split(",")], xi1=int(x1),
                             l2=[None if s == "-" else int(s) for s in l2.split(",")], xi2=int(x2),
                             order=[int(o) for o in order.split()]))
    return rows


def test_toy_hand_trace_cascade_level():
    """Appendix-A hand trace: every branch of Alg. 2 (sink, fill, eager, accept+promote,
    accept+drop, select in, select keep, tie) step by step."""
    rows = _load_toy_trace()
    head = CascadeHead(sink_size=1, cache_size=4, num_cascades=2)
    for row in rows:
        head.add_token(Token(origin=row["t"], mu=row["mu"]))
        l1 = [None if tok is None else tok.origin for tok in head.rings[0].slots]
        l2 = [None if tok is None else tok.origin for tok in head.rings[1].slots]
        assert l1 == row["l1"], row
        assert l2 == row["l2"], row
        assert head.rings[0].xi == row["xi1"] and head.rings[1].xi == row["xi2"], row
        assert [o for o, _ in head.positions()] == row["order"], row
        assert [pe for _, pe in head.positions()] == list(range(len(row["order"])))
    kinds = {e.kind for e in head.events}
    assert {"sink", "fill", "eager", "accept", "select_in", "select_keep", "drop_end"} <= kinds
    # final pe by flat slot: sink->0, L2 s1->1, L2 s0->2, L1 s1->3, L1 s0->4
    cfg = OracleConfig(1, 1, 1, 1, 2, 1, 4, 2, gamma=0.0)
    orc = CascadeOracle(cfg)
    for row in rows:
        s = np.zeros((1, 1, cfg.s_tot + 1))
        st = orc.state(0)
        for x in range(cfg.s_tot):                    # inject each resident's scripted mu
            o = st["origin"][0, 0, x]
            if o >= 0:
                s[0, 0, x] = rows[o]["mu"]
        s[0, 0, cfg.s_tot] = row["mu"]
        orc.update_with_scores(0, np.zeros((1, 1, 1, 2)), np.zeros((1, 1, 1, 2)), s)
    st = orc.state(0)
    assert list(st["origin"][0, 0]) == [0, 11, 10, 8, 7]
    assert list(st["pe"][0, 0]) == [0, 4, 3, 2, 1]


def test_spec_example_s146_selection_keeps_heavy_token():
    """N=2, caps 1/1, alpha=1, score(p3) >> others: after p5, C2 holds p3, C1 holds p5."""
    head = CascadeHead(1, 2, 2)
    for t in range(6):
        head.add_token(Token(origin=t, mu=100.0 if t == 3 else 0.0))
    assert head.rings[0].slots[0].origin == 5
    assert head.rings[1].slots[0].origin == 3


def test_accepting_pattern_matches_paper_rates():
    """sub-cache 1 takes every token, 2 every 2nd iteration, 3 every 4th."""
    assert all(CascadeHead.accepting(1, t) for t in range(16))
    assert [CascadeHead.accepting(2, t) for t in (3, 4)] == [False, True]
    assert [CascadeHead.accepting(3, t) for t in range(8)] == [True, False, False, False] * 2


def test_positional_reindex_paper_example():
    """cache holding stream indices [0,1,3,5,7,8] -> pe [0..5]."""
    m = reindex_positions([0, 1, 3, 5, 7, 8])
    assert [m[o] for o in [0, 1, 3, 5, 7, 8]] == [0, 1, 2, 3, 4, 5]


def test_positional_reindex_example_reached_by_alg2():
    """Find an Alg. 2 run whose residents are exactly {0,1,3,5,7,8} and check their pe."""
    # alpha=2 sinks, N=4 x c=1 (found by exhaustive search over mu in {0,1,2}^9); p3 is heavy.
    found = False
    for mus in [(0, 0, 0, 1, 0, 0, 0, 0, 0)]:
        head = CascadeHead(2, 4, 4)
        for t in range(9):
            head.add_token(Token(origin=t, mu=float(mus[t])))
        origins = [o for o, _ in head.positions()]
        if origins == [0, 1, 3, 5, 7, 8]:
            found = True
            assert [pe for _, pe in head.positions()] == [0, 1, 2, 3, 4, 5]
    assert found, origins


def _random_stream_check(alpha, C, N, T, rng):
    head = CascadeHead(alpha, C, N)
    naive = NaiveCascade(alpha, C, N)
    mus = rng.random(T)
    # quantise some scores to force ties
    mus = np.where(rng.random(T) < 0.2, 0.5, mus)
    for t in range(T):
        head.add_token(Token(origin=t, mu=float(mus[t])))
        naive.add(t, float(mus[t]))
        # two independent models agree on the logical contents and counts
        assert [o for o, _ in head.positions()] == naive.logical_origins()
        assert head.counts() == naive.counts()
        # invariants: capacity, sinks never evicted, ascending origins (age order), uniqueness
        assert sum(head.counts()) <= C and len(head.sink) == min(alpha, t + 1)
        assert [tok.origin for tok in head.sink] == list(range(min(alpha, t + 1)))
        origins = [o for o, _ in head.positions()]
        assert origins == sorted(set(origins))
        for ring in head.rings:
            if not ring.is_full():
                assert ring.xi == ring.count % ring.cap
                assert all(s is None for s in ring.slots[ring.count:])
    return head


def test_ring_vs_naive_random_streams():
    rng = np.random.default_rng(1234)
    n = 0
    for _ in range(1000):
        N = int(rng.integers(1, 5))
        c = int(rng.integers(1, 5))
        alpha = int(rng.integers(0, 4))
        T = int(rng.integers(1, 60))
        _random_stream_check(alpha, N * c, N, T, rng)
        n += 1
    assert n == 1000


def test_single_cascade_is_sink_plus_fifo_window():
    """N=1 is the Streaming-LLM sink cache: first alpha tokens + the last |C| tokens."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        alpha = int(rng.integers(0, 5))
        C = int(rng.integers(1, 9))
        T = int(rng.integers(1, 10 * C + alpha + 1))
        head = CascadeHead(alpha, C, 1)
        for t in range(T):
            head.add_token(Token(origin=t, mu=float(rng.random())))
            expect = list(range(min(alpha, t + 1))) + list(range(max(alpha, t + 1 - C), t + 1))
            assert [o for o, _ in head.positions()] == expect


def _span_run(C, N, T, alpha=0):
    """Keep-resident ties (all mu equal): returns steady-state spans newest-oldest+1."""
    head = CascadeHead(alpha, C, N)
    spans = []
    S_tilde = token_span(C, N)
    for t in range(T):
        head.add_token(Token(origin=t, mu=0.0))
        if t > 4 * S_tilde:
            non_sink = [o for o, _ in head.positions()][len(head.sink):]
            spans.append(non_sink[-1] - non_sink[0] + 1)
    return np.array(spans)


@pytest.mark.parametrize("C,N", [(8, 4), (64, 4), (40, 2), (16, 1), (64, 8)])
def test_eq4_span_is_exact_max(C, N):
    """Eq. 4: the span of the cache window never exceeds S~ and reaches it."""
    S_tilde = token_span(C, N)
    spans = _span_run(C, N, 6 * S_tilde + 200)
    assert spans.max() == S_tilde
    assert spans.min() >= S_tilde - (2 ** (N - 1) - 1)


@pytest.mark.slow
def test_eq4_span_4096_4():
    """SPEC acceptance criterion 2 scale: |C|=4096, N=4 -> S~ = 15360."""
    spans = _span_run(4096, 4, 15360 * 4 + 4000)
    assert spans.max() == 15360 and spans.min() >= 15360 - 7


def test_eq4_and_sparsity_values():
    assert token_span(8, 4) == 30                    # (8/4)*(1+2+4+8)
    assert token_span(4096, 4) == 15360
    assert token_span(17, 1) == 17                   # N=1: sliding window
    ov, win = sparsity(4096, 4, 32768)
    assert ov == pytest.approx(0.875, abs=0) and win == pytest.approx(1 - 4096 / 15360, abs=1e-15)
    assert stride_chunks(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert stride_chunks(4, 8) == [(0, 4)]


@pytest.mark.parametrize("alpha,c,N", [(4, 16, 4), (1, 2, 2), (64, 1024, 4), (3, 5, 3), (64, 8, 8)])
def test_first_drop_position(alpha, c, N):
    """No token is dropped while S <= alpha + 2c; the first drop happens at the first
    t >= alpha + 2c at which sub-cache 2 does not accept (N >= 3) or at alpha + 2c (N = 2)."""
    head = CascadeHead(alpha, N * c, N)
    first = None
    t = 0
    while first is None:
        head.add_token(Token(origin=t, mu=0.0))
        if any(e.kind in ("drop_sel", "drop_end") for e in head.events if e.t == t):
            first = t
        t += 1
    assert first >= alpha + 2 * c
    if N == 2:
        assert first == alpha + 2 * c
    else:
        x = alpha + 2 * c
        expect = x if x % 2 == 1 else x + 1
        assert first == expect


def test_counts_xi_positions_independent_of_scores():
    """Only selection outcomes depend on mu: counts, xi, t and pe never do."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        N, c, alpha = int(rng.integers(1, 5)), int(rng.integers(1, 6)), int(rng.integers(0, 4))
        a, b = CascadeHead(alpha, N * c, N), CascadeHead(alpha, N * c, N)
        for t in range(int(rng.integers(1, 120))):
            a.add_token(Token(t, mu=float(rng.random())))
            b.add_token(Token(t, mu=float(rng.random())))
            assert a.counts() == b.counts() and a.xis() == b.xis()
            assert [pe for _, pe in a.positions()] == [pe for _, pe in b.positions()]


def test_ring_push_and_replace_semantics():
    """SPEC S:39-67 ring examples (push_overwrite / evict_newest / peek_newest)."""
    r = Ring(2)
    assert r.push(Token(0)) is None
    assert r.push(Token(1)) is None
    assert r.push(Token(2)).origin == 0 and [t.origin for t in r.oldest_to_newest()] == [1, 2]
    assert r.newest().origin == 2
    r.replace_newest(Token(3))
    assert [t.origin for t in r.oldest_to_newest()] == [1, 3]
    assert r.push(Token(4)).origin == 1 and r.push(Token(5)).origin == 3


def test_selection_off_is_keep_resident_and_scores_irrelevant():
    """Reading Q3 ("w/o token selection"): the resident stays and the carried token is
    dropped, i.e. the cascade behaves as under score selection with all scores equal (strict
    '>' never fires, Q2).  Pinned three ways on random streams: (1) contents equal those of a
    selection-on cascade fed equal scores, (2) the ring model equals the shifting-list model
    with selection off, (3) the span stays in the keep-resident band [S~ - (2^(N-1) - 1), S~]
    of SURVEY App. B.2 (Eq. 4)."""
    rng = np.random.default_rng(99)
    for _ in range(300):
        N = int(rng.integers(1, 5))
        c = int(rng.integers(1, 5))
        alpha = int(rng.integers(0, 4))
        T = int(rng.integers(1, 80))
        off = CascadeHead(alpha, N * c, N, selection=False)
        tied = CascadeHead(alpha, N * c, N)
        naive = NaiveCascade(alpha, N * c, N, selection=False)
        for t in range(T):
            mu = float(rng.random())
            off.add_token(Token(origin=t, mu=mu))
            tied.add_token(Token(origin=t, mu=0.25))
            naive.add(t, mu)
            got = [o for o, _ in off.positions()]
            assert got == [o for o, _ in tied.positions()]
            assert got == naive.logical_origins()
    for C, N in [(8, 4), (64, 4), (40, 2), (64, 8)]:
        head = CascadeHead(0, C, N, selection=False)
        S_tilde = token_span(C, N)
        spans = []
        for t in range(6 * S_tilde + 200):
            head.add_token(Token(origin=t, mu=float(rng.random())))
            if t > 4 * S_tilde:
                o = [x for x, _ in head.positions()]
                spans.append(o[-1] - o[0] + 1)
        assert max(spans) == S_tilde and min(spans) >= S_tilde - (2 ** (N - 1) - 1)


def test_homogeneous_head_policy():
    """Homogeneous heads: one selection per sequence.  Pins: every kv-head's cascade
    holds the same origins after every chunk; with one kv-head the policy is the independent
    one; under max, each kv-head's s is the max over ALL q-heads, so it bounds every group's
    own max; under mean, the sum rule 1 - gamma^m (Alg. 3) still holds."""
    from oracle.attention import reduce_heads
    rng = np.random.default_rng(21)
    d, m = 16, 12
    base = dict(num_layers=1, batch=2, head_dim=d, sink_size=2, cache_size=8, num_cascades=4,
                gamma=0.9)
    for how in ("max", "mean"):
        hom = CascadeOracle(OracleConfig(num_q_heads=8, num_kv_heads=4, head_policy="homogeneous",
                                         head_reduce=how, **base))
        for _ in range(6):
            q = rng.standard_normal((2, m, 8, d))
            k, v = rng.standard_normal((2, m, 4, d)), rng.standard_normal((2, m, 4, d))
            _, s, s_heads = hom.prefill_stride(0, q, k, v, return_heads=True)
            st = hom.state(0)
            for b in range(2):
                assert all(np.array_equal(st["origin"][b, 0], st["origin"][b, g]) for g in range(4))
                assert all(np.array_equal(s[b, 0], s[b, g]) for g in range(4))
                if how == "max":
                    assert np.all(s[b, 0] >= reduce_heads(s_heads[b], 2, "max") - 0)
                else:
                    assert s[b, 0].sum() == pytest.approx(1 - 0.9 ** m, rel=1e-12)
    one = [CascadeOracle(OracleConfig(num_q_heads=3, num_kv_heads=1, head_policy=pol, **base))
           for pol in ("homogeneous", "independent")]
    for _ in range(5):
        q = rng.standard_normal((2, m, 3, d))
        k, v = rng.standard_normal((2, m, 1, d)), rng.standard_normal((2, m, 1, d))
        outs = [o.prefill_stride(0, q, k, v) for o in one]
        np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(one[0].state(0)["origin"], one[1].state(0)["origin"])
