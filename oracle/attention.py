"""Attention with exact per-key EMA mass -- oracle, test infra only (float64).

* ``attention``   Eq. 1: softmax(Q K^T / sqrt(d)) V, exact softmax.
* ``chunk_attention``  the rectangular slice of Fig. 4: the m chunk
  queries attend to all n_c cached keys plus the chunk's own keys causally
  (reading Q10: the cache as it was *before* the chunk).  With m = 1 this is
  Eq. 2.
* ``rope``  rotary encoding applied by cache rank pe, rotate-half
  pairing (i, i + d/2), inverse frequencies theta**(-2i/d), angles in float64
  (reading Q11).
* ``ema_weights`` / ``key_mass``  Alg. 3 in its exact-normaliser
  reading (Q6): row r of a chunk of m queries is one EMA timestep with
  coefficient C_EMA = (1 - gamma) * gamma**k, k = m - (r + 1), and the
  column sum over rows of P weighted by C_EMA is the key's mass s.
  Heads are independent per KV group and reduced with max (Q7).
* ``key_mass_onepass``  Alg. 3 as the paper writes it, in its tile
  order: the normaliser of the column sum at inner step j is the running row sum
  extrapolated over the remaining steps, l_i + l_i * rho / gamma (reading
  Q6b: gamma = inner steps completed including step j, rho = steps remaining).
"""

from __future__ import annotations

import numpy as np


def inv_freq(d: int, theta: float) -> np.ndarray:
    return theta ** (-(np.arange(0, d, 2, dtype=np.float64)) / d)


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """Rotate rows of x[..., n, d] by positions pos[n] (rotate-half convention)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv_freq(d, theta)[None, :]
    cos, sin = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), via float32 -- returned as float64.

    bfloat16 is the top 16 bits of an IEEE float32; rounding adds 0x7fff plus the lowest
    kept bit before truncating the low 16 bits (round-to-nearest-even)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    mx = np.max(logits, axis=-1, keepdims=True)
    e = np.exp(logits - mx)
    return e / np.sum(e, axis=-1, keepdims=True)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, causal: bool,
              scale: float | None = None) -> np.ndarray:
    """Eq. 1 for one head: q [S, d], k [S, d], v [S, d]."""
    d = q.shape[-1]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    logits = (q @ k.T) * scale
    if causal:
        S = q.shape[0]
        logits = np.where(np.tril(np.ones((S, k.shape[0]), dtype=bool)), logits, -np.inf)
    return softmax_rows(logits) @ v


def chunk_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, n_cached: int,
                    scale: float):
    """One head of the strided-prefill slice.

    q [m, d] (already rotated), k/v [n_cached + m, d] (keys rotated): rows
    [0, n_cached) are the cache, rows n_cached + r are the chunk's own keys.
    Query r sees every cached key and chunk keys r' <= r.  Returns (O [m, d],
    P [m, n_cached + m]) with masked entries of P exactly 0.
    """
    m = q.shape[0]
    n = k.shape[0]
    assert n == n_cached + m
    logits = (q @ k.T) * scale
    r = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    visible = j <= n_cached + r
    logits = np.where(visible, logits, -np.inf)
    P = softmax_rows(logits)
    return P @ v, P


def slice_rows(q_rows: np.ndarray, rows: np.ndarray, k: np.ndarray, v: np.ndarray, n_cached: int,
               scale: float):
    """Rows `rows` of the same rectangular slice as ``chunk_attention`` (query r sees keys
    j <= n_cached + r), evaluated for a subset of rows only -- so a long chunk can be checked
    block by block.  Returns (O [len(rows), d], P [len(rows), n_keys])."""
    logits = (q_rows @ k.T) * scale
    visible = np.arange(k.shape[0])[None, :] <= n_cached + np.asarray(rows)[:, None]
    P = softmax_rows(np.where(visible, logits, -np.inf))
    return P @ v, P


def ema_weights(m: int, gamma: float) -> np.ndarray:
    """C_EMA for rows r = 0..m-1: (1 - gamma) * gamma**(m - (r + 1))."""
    k = m - (np.arange(m) + 1)
    return (1.0 - gamma) * np.power(gamma, k.astype(np.float64))


def key_mass(P: np.ndarray, gamma: float) -> np.ndarray:
    """s[j] = sum_r C_EMA[r] * P[r, j]  -- Alg. 3's column sum, exact normaliser."""
    return ema_weights(P.shape[0], gamma) @ P


def reduce_heads(s_heads: np.ndarray, group: int, how: str = "max") -> np.ndarray:
    """Independent head policy: reduce each GQA group of q-heads to its kv-head.

    s_heads [Hq, n] -> [Hq // group, n]."""
    Hq, n = s_heads.shape
    g = s_heads.reshape(Hq // group, group, n)
    if how == "max":
        return g.max(axis=1)
    if how == "mean":
        return g.mean(axis=1)
    if how == "median":
        return np.median(g, axis=1)
    raise ValueError(how)


def gamma_pow(gamma: float, m: int) -> float:
    """gamma**m by right-to-left binary exponentiation in float64.

    The decay applied to mu over a chunk of m rows (P:154 iterated m times, Q4).
    Written out so the product order is fixed (the GPU side documents the same
    order in include/cascade.h)."""
    result = 1.0
    base = float(gamma)
    e = int(m)
    while e > 0:
        if e & 1:
            result = result * base
        base = base * base
        e >>= 1
    return result


def key_mass_onepass(q_rot: np.ndarray, k_rot: np.ndarray, n_cached: int, scale: float, gamma: float,
                     key_tiles, q_tile: int = 128):
    """Alg. 3 step by step, in the order of its two loops.

    q_rot [m, d]; k_rot [n_cached + m, d] (rows [0, n_cached) the cache, n_cached + r the
    chunk's keys).  key_tiles: the cache's key tiles in loop order, each a list of row indices
    into k_rot; the chunk's own keys follow as tiles of q_tile keys (a query block sees the chunk
    tiles up to its own, causally masked inside the diagonal one).  For query block i and inner
    step j over its n_i visible key tiles:
        S_ij = Q_i K_j^T * scale                                  (masked entries -inf)
        m_i  = max(m_i, rowmax S_ij);  l_i = l_i exp(m_old - m_i) + rowsum exp(S_ij - m_i)
        S^_ij = exp(S_ij - m_i)                                   (max-adjusted, unnormalised)
        C_EMA = (1 - gamma) gamma^(m - (r + 1)) per query row r
        score[K_j] += col_sum( S^_ij / (l_i + l_i rho / gamma_) * C_EMA ),
            gamma_ = j + 1 (steps completed), rho = n_i - (j + 1) (steps remaining)
    Returns s [n_cached + m]."""
    m = q_rot.shape[0]
    s = np.zeros(k_rot.shape[0])
    c_ema = ema_weights(m, gamma)
    chunk_tiles = [list(range(n_cached + t0, n_cached + min(m, t0 + q_tile))) for t0 in range(0, m, q_tile)]
    for i0 in range(0, m, q_tile):
        rows = np.arange(i0, min(m, i0 + q_tile))
        tiles = list(key_tiles) + chunk_tiles[: i0 // q_tile + 1]
        n_i = len(tiles)
        m_i = np.full(len(rows), -np.inf)
        l_i = np.zeros(len(rows))
        for j, cols in enumerate(tiles):
            cols = np.asarray(cols)
            S = (q_rot[rows] @ k_rot[cols].T) * scale
            S = np.where(cols[None, :] <= n_cached + rows[:, None], S, -np.inf)   # causal in the chunk
            m_new = np.maximum(m_i, S.max(axis=1))
            l_i = l_i * np.exp(m_i - m_new) + np.exp(S - m_new[:, None]).sum(axis=1)
            m_i = m_new
            S_hat = np.exp(S - m_i[:, None])
            gamma_, rho = j + 1, n_i - (j + 1)
            s[cols] += ((S_hat / (l_i + l_i * rho / gamma_)[:, None]) * c_ema[rows][:, None]).sum(axis=0)
    return s
