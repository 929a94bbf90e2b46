"""CPU tests of the C ABI: the library loads, exports every symbol include/cascade.h declares,
validates configs, and its host mirror (the schedule every kernel launch is built from)
reproduces the oracle's Alg. 2 counters and positions exactly."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle.cascade import CascadeHead, Token
from paper_2406_17808_b200 import cascade as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "cascade.h")).read()
    return sorted(set(re.findall(r"\b(cascade_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = C.lib()
    declared = _declared_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(L, name), name
    assert set(C.EXPORTED) == set(declared)


def test_status_strings():
    L = C.lib()
    for code in range(0, -8, -1):
        assert L.cascade_status_string(code)


@pytest.mark.parametrize("field,value,code", [
    ("cache_size", 4097, -2), ("num_cascades", 0, -2), ("num_q_heads", 30, -2),
    ("head_dim", 96, -2), ("ema_gamma", 1.5, -2), ("max_stride", 0, -2), ("num_cascades", 17, -2)])
def test_config_validation(field, value, code):
    cfg = C.CascadeConfig()
    assert C.validate(cfg) == 0
    setattr(cfg, field, value)
    assert C.validate(cfg) == code
    assert C.workspace_bytes(cfg) == 0


def test_ablation_options_validate():
    """head_reduce 0/1/2 (max, mean, median: P:542) and selection 0/1 (Q3) are accepted; others are
    CONFIG errors; head_policy 0/1 (independent, homogeneous: P:542); the median over all heads of a
    sequence needs Hq <= 32 (UNSUPPORTED above)."""
    import ctypes
    L = C.lib()
    assert C.validate(C.CascadeConfig(head_reduce="mean", selection=False)) == 0
    assert C.validate(C.CascadeConfig(head_reduce="median")) == 0
    assert C.validate(C.CascadeConfig(head_reduce="median", num_q_heads=33, num_kv_heads=1, dtype="f32")) == -7
    assert C.validate(C.CascadeConfig(num_q_heads=32, num_kv_heads=2)) == -7      # bf16 group 16
    assert C.validate(C.CascadeConfig(num_q_heads=32, num_kv_heads=2, dtype="f32")) == 0
    assert C.validate(C.CascadeConfig(head_policy="homogeneous", head_reduce="mean")) == 0
    assert C.validate(C.CascadeConfig(head_policy="homogeneous", head_reduce="median")) == 0
    assert C.validate(C.CascadeConfig(head_policy="homogeneous", head_reduce="median", num_q_heads=64,
                                      num_kv_heads=8)) == -7
    for field, value, code in [("head_reduce", 3, -2), ("selection", 2, -2), ("head_policy", 2, -2)]:
        st = C.CascadeConfig().c_struct()
        setattr(st, field, value)
        assert L.cascade_validate_config(ctypes.byref(st)) == code


def test_workspace_bytes_grow_with_layers():
    a = C.workspace_bytes(C.CascadeConfig(num_layers=1))
    b = C.workspace_bytes(C.CascadeConfig(num_layers=2))
    assert 0 < a < b


def _oracle_pe(head, alpha, N, c):
    pe = np.full(alpha + N * c, -1, dtype=np.int32)
    rank = {id(t): p for p, t in enumerate(head.logical_order())}
    for s, tok in enumerate(head.sink):
        pe[s] = rank[id(tok)]
    for i, ring in enumerate(head.rings):
        for s, tok in enumerate(ring.slots):
            if tok is not None:
                pe[alpha + i * c + s] = rank[id(tok)]
    return pe


def test_host_mirror_matches_oracle_counters_and_positions():
    rng = np.random.default_rng(99)
    for _ in range(150):
        N = int(rng.integers(1, 6))
        c = int(rng.integers(1, 9))
        alpha = int(rng.integers(0, 6))
        sel = bool(rng.random() < 0.7)
        cfg = C.CascadeConfig(sink_size=alpha, cache_size=N * c, num_cascades=N, max_stride=64,
                              selection=sel)
        mirror = C.Mirror()
        head = CascadeHead(alpha, N * c, N, selection=sel)
        T = 0
        for _ in range(int(rng.integers(1, 12))):
            m = int(rng.integers(1, 40))
            pe, ops = C.mirror_advance(cfg, mirror, m)
            drops_before = sum(1 for e in head.events if e.kind in ("drop_sel", "drop_end"))
            for t in range(T, T + m):
                head.add_token(Token(t, mu=float(rng.random())))
            T += m
            drops = sum(1 for e in head.events if e.kind in ("drop_sel", "drop_end")) - drops_before
            assert mirror.t == T
            assert mirror.sink_count == len(head.sink)
            assert list(mirror.counts[:N]) == head.counts()
            assert list(mirror.xi[:N]) == head.xis()
            np.testing.assert_array_equal(pe, _oracle_pe(head, alpha, N, c))
            assert ops[2] == drops
            assert ops[3] in (0, 1) or m > c       # selections of a chunk are independent unless m > c
            if not sel:
                assert ops[0] == 0 and ops[3] == 0  # no selection: nothing to resolve on the device


def test_cfg3_schedule_is_depth_zero_and_fill_trajectory():
    """cfg3 (N=8, c=8192, m=4096): every selection of every chunk is resolvable in one pass, and
    the cache never fills within 2^20 tokens."""
    cfg = C.CascadeConfig(sink_size=64, cache_size=65536, num_cascades=8, max_stride=4096)
    mirror = C.Mirror()
    for _ in range(256):
        pe, ops = C.mirror_advance(cfg, mirror, 4096, want_pe=False)
        assert ops[3] <= 1
    assert mirror.t == 1 << 20
    assert sum(mirror.counts[:8]) < 65536


def test_binding_fails_loudly_without_the_library(monkeypatch, tmp_path):
    """No CPU fallback: with the shared library absent the binding raises instead of computing
    anything elsewhere (the product path must fail loudly)."""
    monkeypatch.setattr(C, "_lib", None)
    monkeypatch.setattr(C, "LIB_PATH", str(tmp_path / "libcascade.so"))
    with pytest.raises(RuntimeError, match="missing"):
        C.lib()
    with pytest.raises(RuntimeError, match="missing"):
        C.validate(C.CascadeConfig())
