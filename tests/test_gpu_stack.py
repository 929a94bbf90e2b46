"""GPU parity of the coupled layer stack (cascade_stack: Alg. 1's layer
loop) through the C ABI:

* the wavefront (all chunks enqueued at once, layers of consecutive chunks overlapping on their
  streams) is bit-identical to running the chunks one call at a time;
* every layer of every chunk against the oracle given the same layer inputs: the projections
  (q, k, v = x W; x_out = x + o W_o) against float64 products of the GPU's bf16 operands, and the
  layer's attention, exact per-key mass and cascade contents against ``CascadeOracle`` fed the
  GPU's q, k, v (selection margins audited above 1e-3);
* below the first drop, the whole stack against the float64 stack oracle (``oracle.stack``).
"""

import numpy as np
import pytest
import torch

from oracle.model import CascadeOracle, OracleConfig
from oracle.stack import StackOracle, stack_config
from paper_2406_17808_b200 import cascade as C

pytestmark = pytest.mark.gpu

L, B, HQ, HK, D_HEAD, D_MODEL = 3, 2, 4, 2, 64, 256


def _np(t):
    return t.detach().to("cpu", torch.float64).numpy()


def _bf(a):
    return torch.from_numpy(np.asarray(a)).to(torch.bfloat16)


def _weights(seed, qk_scale=3.0):
    """Per layer (w_q, w_k, w_v, w_o) as bf16 values; q/k scaled up so attention is peaked
    (selection margins, SURVEY 8(d) margin audit: seed 33 gives a minimum relative margin of
    3.0e-3 over 1896 selections in the float64 stack), v and o scaled down so the residual stream
    and the outputs stay at unit scale, where the north star's 2e-2 bf16 tolerance applies."""
    rng = np.random.default_rng(seed)
    s = 1.0 / np.sqrt(D_MODEL)
    shapes = [(D_MODEL, HQ * D_HEAD), (D_MODEL, HK * D_HEAD), (D_MODEL, HK * D_HEAD), (HQ * D_HEAD, D_MODEL)]
    scales = [qk_scale * s, qk_scale * s, 0.5 * s, 0.5 * s]
    ws = [[_bf(rng.standard_normal(sh) * sc) for sh, sc in zip(shapes, scales)] for _ in range(L)]
    return ws, rng


def _cfg(cache=96, N=3, sinks=4, m=32):
    return C.CascadeConfig(num_layers=L, batch=B, num_q_heads=HQ, num_kv_heads=HK, head_dim=D_HEAD,
                           sink_size=sinks, cache_size=cache, num_cascades=N, max_stride=m, dtype="bf16",
                           rope_theta=10000.0)


def _stack(cfg, ws):
    cas = C.Cascade(cfg)
    dev = [tuple(w.cuda() for w in lw) for lw in ws]
    return cas, C.Stack(cas, dev, D_MODEL)


def _states_equal(a, b):
    for l in range(L):
        sa, sb = a.state(l), b.state(l)
        for key in ("origin", "mu", "pe"):
            assert torch.equal(sa[key], sb[key]), (l, key)
        assert torch.equal(sa["k"].view(torch.int16), sb["k"].view(torch.int16)), l
        assert (sa["t"], sa["counts"], sa["xi"]) == (sb["t"], sb["counts"], sb["xi"])


def test_stack_wavefront_bit_identical_to_one_chunk_per_call():
    cfg = _cfg()
    ws, rng = _weights(33)
    T, m = 300, 32
    x = _bf(rng.standard_normal((B, T, D_MODEL))).cuda()
    cas_a, st_a = _stack(cfg, ws)
    ya = st_a.prefill(x, m)
    cas_b, st_b = _stack(cfg, ws)
    yb = torch.empty_like(x)
    for a in range(0, T, m):
        xb = x[:, a:a + m].contiguous()
        yb[:, a:a + m] = st_b.prefill(xb, m)
    torch.cuda.synchronize()
    assert torch.equal(ya.view(torch.int16), yb.view(torch.int16))
    _states_equal(cas_a, cas_b)


def _per_layer_run(seed, T=240, m=32):
    """One seeded stack run checked layer by layer against the oracle fed the GPU's own layer
    inputs.  Returns (first failure or None, oracle margins, stats)."""
    cfg = _cfg()
    ws, rng = _weights(seed)
    x = _bf(rng.standard_normal((B, T, D_MODEL))).cuda()
    cas, st = _stack(cfg, ws)
    orc = CascadeOracle(OracleConfig(L, B, HQ, HK, D_HEAD, cfg.sink_size, cfg.cache_size, cfg.num_cascades,
                                     gamma=cfg.ema_gamma, rope_theta=cfg.rope_theta, round_operands="bf16"))
    W = [[_np(w) for w in lw] for lw in ws]
    worst_proj, worst_o = 0.0, 0.0
    try:
        for a in range(0, T, m):
            mm = min(m, T - a)
            st.prefill(x[:, a:a + mm].contiguous(), m)
            torch.cuda.synchronize()
            prev_out = None
            for l in range(L):
                tr = {k: _np(v) for k, v in st.trace(l).items()}
                if l == 0:
                    np.testing.assert_array_equal(tr["x_in"], _np(x[:, a:a + mm]))
                else:                               # layer l consumes layer l-1's output of this chunk
                    np.testing.assert_array_equal(tr["x_in"], prev_out)
                xi = tr["x_in"].reshape(B * mm, D_MODEL)
                for key, w, H in (("q", W[l][0], HQ), ("k", W[l][1], HK), ("v", W[l][2], HK)):
                    ref = (xi @ w).reshape(B, mm, H, D_HEAD)
                    err = np.abs(tr[key] - ref).max() / np.abs(ref).max()
                    worst_proj = max(worst_proj, err)
                    assert err < 1e-2, (a, l, key, err)   # bf16 output rounding (2^-9) + fp32 accumulation
                O_ref, s_ref = orc.prefill_stride(l, tr["q"], tr["k"], tr["v"])
                worst_o = max(worst_o, np.abs(tr["o"] - O_ref).max())
                assert np.abs(tr["o"] - O_ref).max() <= 2e-2, (a, l)
                np.testing.assert_allclose(_np(cas.last_scores(l)), s_ref, rtol=1e-3, atol=1e-30)
                g, o_st = cas.state(l), orc.state(l)
                np.testing.assert_array_equal(g["origin"].cpu().numpy(), o_st["origin"])
                np.testing.assert_array_equal(g["k"].double().cpu().numpy()[o_st["origin"] >= 0],
                                              o_st["k"][o_st["origin"] >= 0])
                ref = xi + tr["o"].reshape(B * mm, -1) @ W[l][3]
                err = np.abs(tr["x_out"].reshape(B * mm, -1) - ref).max() / np.abs(ref).max()
                assert err < 1e-2, (a, l, err)
                prev_out = tr["x_out"]
        failure = None
    except AssertionError as e:
        failure = e
    return failure, orc.select_margins(), (worst_proj, worst_o)


def test_stack_every_layer_matches_oracle_given_its_inputs():
    """Margin audit: a run counts only if every selection the oracle takes on the
    GPU's layer inputs has relative margin > 1e-3; otherwise the seed advances by +7 (logged) --
    the layer inputs are the GPU's own bf16 GEMM outputs, so the audit cannot be settled on the
    host beforehand.  A failure in an audited run is a failure."""
    # seeds 33, 40, 47, 54, 61 ran before this start point (minimum margins 8.7e-4, 4.8e-4, 6.4e-4,
    # 8.3e-4, 9.6e-4 -- and every state check passed on each); 68 passed the audit (1.5e-3)
    seed, log = 68, []
    for _ in range(8):
        failure, margins, (wp, wo) = _per_layer_run(seed)
        ok = margins.size > 0 and margins.min() > 1e-3
        log.append((seed, int(margins.size), float(margins.min()) if margins.size else None, failure is None))
        if ok:
            if failure is not None:
                raise failure
            print(f"stack: seeds {log}; worst projection rel err {wp:.2e}, worst |dO| {wo:.2e}")
            return
        seed += 7
    pytest.fail(f"no seed passed the margin audit: {log}")


def test_stack_below_first_drop_matches_float64_stack_oracle():
    """alpha 4, |C| 96, N 3: no token leaves before t = alpha + 2c = 68 (App. B.3); 64 tokens in
    strides of 16 through the stack vs the float64 stack oracle (bf16 rounding of the
    intermediates at the GPU's points, reading Q22), end to end."""
    cfg = _cfg(m=16)
    ws, rng = _weights(7, qk_scale=1.0)
    T = 64
    x = _bf(rng.standard_normal((B, T, D_MODEL)))
    cas, st = _stack(cfg, ws)
    y = _np(st.prefill(x.cuda(), 16))
    orc = StackOracle(stack_config(L, B, HQ, HK, D_HEAD, 4, 96, 3, rope_theta=10000.0, round_operands="bf16"),
                      *[[_np(lw[i]) for lw in ws] for i in range(4)], round_bf16_io=True)
    ref = np.concatenate([orc.prefill_stride(_np(x[:, a:a + 16])) for a in range(0, T, 16)], axis=1)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    assert err < 2e-2, err
    for l in range(L):
        org = cas.state(l)["origin"].cpu().numpy()
        assert sorted(org[org >= 0].tolist()) == sorted(list(range(T)) * (B * HK))


def test_stack_rejects_bad_inputs():
    cfg = _cfg()
    ws, _ = _weights(1)
    cas = C.Cascade(cfg)
    dev = [tuple(w.cuda() for w in lw) for lw in ws]
    with pytest.raises(ValueError):
        C.Stack(cas, dev[:2], D_MODEL)
    st = C.Stack(cas, dev, D_MODEL)
    with pytest.raises(ValueError):
        st.prefill(torch.zeros((B, 10, D_MODEL + 1), dtype=torch.bfloat16, device="cuda"), 8)
    with pytest.raises(C.CascadeError):
        st.prefill(torch.zeros((B, 10, D_MODEL), dtype=torch.bfloat16, device="cuda"), cfg.max_stride + 1)


def test_stack_host_buffers_and_ragged_length_match_device_run():
    """x / y in pinned host memory (the chunk gather / scatter are 2-D host<->device copies inside
    the library) and a length that is not a multiple of the stride: bit-identical to the run on
    device buffers."""
    cfg = _cfg()
    ws, rng = _weights(5)
    T, m = 77, 32
    x = _bf(rng.standard_normal((B, T, D_MODEL)))
    _, st_d = _stack(cfg, ws)
    y_dev = st_d.prefill(x.cuda(), m)
    _, st_h = _stack(cfg, ws)
    xh = x.pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    st_h.prefill(xh, m, yh)
    torch.cuda.synchronize()
    assert torch.equal(yh.view(torch.int16), y_dev.cpu().view(torch.int16))
