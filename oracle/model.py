"""Alg. 1 strided prefill + decode over a cascade per (layer, sequence, kv-head) -- oracle, test infra only.

Per call, for one layer (Alg. 1; cache.get -> layer -> cache.update):

 1. Logical order of the residents = sinks, then C_N ... C_1 oldest -> newest;
    resident p gets pe = p and chunk token r gets pe = n_c + r.
 2. RoPE by pe on cached keys, chunk keys and chunk queries (Q11).
 3. For every q-head h of kv-group g = h // G: exact chunk attention (Eq. 1/2,
    Fig. 4 slice) and its per-key EMA mass s_h (Alg. 3, exact normaliser, Q6).
 4. s_g = max_h s_h over the group (independent heads + max, Q7); the head-reduction
    ablation takes the mean or the median instead (``head_reduce``); the homogeneous
    head policy reduces over all q-heads of the sequence instead (``head_policy``).
 5. Fold (P:154 over m rows, Q4): residents mu <- gamma**m * mu + s_g;
    chunk tokens start at mu = 0, so mu = s_g (Q8).  All folds happen before
    any insertion (Q9).
 6. Insert chunk tokens r = 0..m-1 in order with Alg. 2 (``oracle.cascade``).

Flat slot space (the interface both sides agree on):
sink slot s -> s;  ring slot s of sub-cache i (1-indexed) -> alpha + (i-1)*c + s;
chunk row r -> S_tot + r, S_tot = alpha + |C|.  Scores s and the exported state
are indexed in this space; empty slots have score 0, origin -1, pe -1.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List

import numpy as np

from .attention import chunk_attention, gamma_pow, key_mass, key_mass_onepass, reduce_heads, rope, round_bf16
from .cascade import CascadeHead, Token


@dataclass
class OracleConfig:
    num_layers: int
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    sink_size: int
    cache_size: int
    num_cascades: int
    gamma: float = 0.9999
    rope_theta: float = 10000.0
    softmax_scale: float = 0.0        # 0 -> 1/sqrt(d)
    selection: bool = True            # False: the ablation without token selection (Q3)
    head_reduce: str = "max"          # GQA reduction of s: "max" (the paper's), "mean", "median"
    # head policy: "independent" (each kv-head's cascade decides on its group's s_g, the
    # paper's choice) or "homogeneous" (one decision per sequence: s reduced over ALL q-heads
    # and applied to every kv-head, whose cascades then hold the same tokens)
    head_policy: str = "independent"
    # Reading Q17: in the bf16 configs the rotated q and k are the operands the score
    # products consume, held in bf16 (the model dtype the paper's kernel runs in); the
    # oracle rounds them to bf16 (round-to-nearest-even) before its float64 dot products.
    round_operands: str = ""          # "" or "bf16"
    # per-key mass (Alg. 3): "exact" (reading Q6: the final LSE, two passes) or "onepass" (the
    # paper's own estimator, in the tile order of ``key_mass_onepass``: the cache's
    # occupied runs in flat-slot order -- sinks, then sub-caches 1..N -- cut into `tile`-slot
    # tiles, then the chunk's keys in tiles of `tile`).  Decode steps (``decode``) keep the exact
    # mass in both modes (the single-token kernel knows the final LSE before it writes a mass).
    score_mode: str = "exact"
    tile: int = 128

    @property
    def c(self) -> int:
        return self.cache_size // self.num_cascades

    @property
    def s_tot(self) -> int:
        return self.sink_size + self.cache_size

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def scale(self) -> float:
        return self.softmax_scale if self.softmax_scale > 0 else 1.0 / np.sqrt(self.head_dim)


class CascadeOracle:
    def __init__(self, cfg: OracleConfig):
        if cfg.num_q_heads % cfg.num_kv_heads:
            raise ValueError("Hq % Hkv != 0")
        self.cfg = cfg
        self.heads: List[List[List[CascadeHead]]] = [
            [[CascadeHead(cfg.sink_size, cfg.cache_size, cfg.num_cascades, cfg.selection)
              for _ in range(cfg.num_kv_heads)] for _ in range(cfg.batch)]
            for _ in range(cfg.num_layers)]

    # ------------------------------------------------------------------ helpers
    def _flat_slots(self, head: CascadeHead) -> Dict[int, Token]:
        """Map flat slot -> resident token."""
        cfg = self.cfg
        out = {}
        for s, tok in enumerate(head.sink):
            out[s] = tok
        for i, ring in enumerate(head.rings):
            for s, tok in enumerate(ring.slots):
                if tok is not None:
                    out[cfg.sink_size + i * cfg.c + s] = tok
        return out

    def _fold_and_insert(self, head: CascadeHead, k_rows, v_rows, s_flat: np.ndarray) -> None:
        cfg = self.cfg
        m = k_rows.shape[0]
        g_m = gamma_pow(cfg.gamma, m)
        for x, tok in self._flat_slots(head).items():           # fold residents first (Q9)
            tok.mu = g_m * tok.mu + float(s_flat[x])
        t0 = head.t
        for r in range(m):                                       # then insert in order
            mu_new = 0.0 * g_m + float(s_flat[cfg.s_tot + r])    # mu starts at 0 (Q8)
            head.add_token(Token(origin=t0 + r, k=np.array(k_rows[r], dtype=np.float64),
                                 v=np.array(v_rows[r], dtype=np.float64), mu=mu_new))

    # ------------------------------------------------------------------ API
    def _key_tiles(self, head: CascadeHead, key_slot) -> list:
        """The cache's key tiles for the one-pass estimator, as row indices of the logical-order
        key array: each occupied run of flat slots (sinks, sub-cache 1, ..., sub-cache N) cut
        into tiles of cfg.tile consecutive slots from the run's start."""
        cfg = self.cfg
        row_of = {x: r for r, x in enumerate(key_slot) if x < cfg.s_tot}
        runs = [(0, len(head.sink))] + [(cfg.sink_size + i * cfg.c, ring.count)
                                        for i, ring in enumerate(head.rings)]
        tiles = []
        for start, n in runs:
            for o in range(0, n, cfg.tile):
                tiles.append([row_of[start + x] for x in range(o, min(n, o + cfg.tile))])
        return tiles

    def prefill_stride(self, layer: int, q: np.ndarray, k: np.ndarray, v: np.ndarray,
                       return_heads: bool = False, exact_mass: bool = False):
        """One Alg. 1 step. q [B,m,Hq,d], k/v [B,m,Hkv,d] (pre-RoPE). Returns (O [B,m,Hq,d], s [B,Hkv,S_tot+m])."""
        cfg = self.cfg
        B, m, Hq, d = q.shape
        G = cfg.group
        O = np.zeros((B, m, Hq, d), dtype=np.float64)
        s_out = np.zeros((B, cfg.num_kv_heads, cfg.s_tot + m), dtype=np.float64)
        s_heads_out = np.zeros((B, Hq, cfg.s_tot + m), dtype=np.float64)
        for b in range(B):
            for g in range(cfg.num_kv_heads):
                head = self.heads[layer][b][g]
                residents = head.logical_order()
                n_c = len(residents)
                flat = {id(tok): x for x, tok in self._flat_slots(head).items()}
                key_slot = [flat[id(tok)] for tok in residents] + [cfg.s_tot + r for r in range(m)]
                kc = [tok.k for tok in residents]
                vc = [tok.v for tok in residents]
                k_all = np.concatenate([np.array(kc).reshape(n_c, d),
                                        np.asarray(k[b, :, g], np.float64)], axis=0)
                v_all = np.concatenate([np.array(vc).reshape(n_c, d),
                                        np.asarray(v[b, :, g], np.float64)], axis=0)
                k_rot = rope(k_all, np.arange(n_c + m), cfg.rope_theta)
                if cfg.round_operands == "bf16":
                    k_rot = round_bf16(k_rot)
                s_h = np.zeros((G, n_c + m))
                for j in range(G):
                    h = g * G + j
                    q_rot = rope(np.asarray(q[b, :, h], np.float64), n_c + np.arange(m), cfg.rope_theta)
                    if cfg.round_operands == "bf16":
                        q_rot = round_bf16(q_rot)
                    o_h, P = chunk_attention(q_rot, k_rot, v_all, n_c, cfg.scale)
                    O[b, :, h] = o_h
                    if cfg.score_mode == "exact" or exact_mass:
                        s_h[j] = key_mass(P, cfg.gamma)
                    elif cfg.score_mode == "onepass":
                        s_h[j] = key_mass_onepass(q_rot, k_rot, n_c, cfg.scale, cfg.gamma,
                                                  self._key_tiles(head, key_slot), cfg.tile)
                    else:
                        raise ValueError(cfg.score_mode)
                    s_heads_out[b, h, key_slot] = s_h[j]
                s_g = reduce_heads(s_h, G, cfg.head_reduce)[0]
                s_out[b, g, key_slot] = s_g
            if cfg.head_policy == "homogeneous":            # one s per sequence
                s_out[b, :] = reduce_heads(s_heads_out[b], Hq, cfg.head_reduce)[0]
            elif cfg.head_policy != "independent":
                raise ValueError(cfg.head_policy)
            for g in range(cfg.num_kv_heads):               # heads' attention all used the pre-chunk state
                self._fold_and_insert(self.heads[layer][b][g], k[b, :, g], v[b, :, g], s_out[b, g])
        if return_heads:
            return O, s_out, s_heads_out
        return O, s_out

    def decode(self, layer: int, q: np.ndarray, k: np.ndarray, v: np.ndarray):
        """Eq. 2 + update: the m = 1 case. q [B,Hq,d], k/v [B,Hkv,d]."""
        O, s = self.prefill_stride(layer, q[:, None], k[:, None], v[:, None], exact_mass=True)
        return O[:, 0], s

    def update_with_scores(self, layer: int, k: np.ndarray, v: np.ndarray, s_flat: np.ndarray) -> None:
        """Score injection: fold the given s [B,Hkv,S_tot+m] and insert k/v [B,m,Hkv,d]."""
        cfg = self.cfg
        if cfg.head_policy == "homogeneous" and cfg.head_reduce == "median":
            # the median of all q-heads is not a function of the kv-head scores given here
            raise ValueError("homogeneous + median needs per-q-head masses; score injection has per-kv-head s")
        s_flat = np.asarray(s_flat, dtype=np.float64)
        for b in range(cfg.batch):
            s_b = s_flat[b]
            if cfg.head_policy == "homogeneous":            # the kv-heads' s reduced per sequence
                s_b = np.broadcast_to(reduce_heads(s_b, cfg.num_kv_heads, cfg.head_reduce), s_b.shape)
            for g in range(cfg.num_kv_heads):
                self._fold_and_insert(self.heads[layer][b][g], k[b, :, g], v[b, :, g], s_b[g])

    def state(self, layer: int) -> dict:
        """Flat-slot export of every (b, g) cascade of a layer."""
        cfg = self.cfg
        B, Hk, S, d = cfg.batch, cfg.num_kv_heads, cfg.s_tot, cfg.head_dim
        origin = np.full((B, Hk, S), -1, dtype=np.int64)
        mu = np.zeros((B, Hk, S), dtype=np.float64)
        pe = np.full((B, Hk, S), -1, dtype=np.int32)
        kr = np.zeros((B, Hk, S, d))
        vv = np.zeros((B, Hk, S, d))
        meta = []
        for b in range(B):
            row = []
            for g in range(Hk):
                head = self.heads[layer][b][g]
                slots = self._flat_slots(head)
                rank = {id(tok): p for p, tok in enumerate(head.logical_order())}
                for x, tok in slots.items():
                    origin[b, g, x] = tok.origin
                    mu[b, g, x] = tok.mu
                    pe[b, g, x] = rank[id(tok)]
                    kr[b, g, x] = tok.k
                    vv[b, g, x] = tok.v
                row.append(dict(t=head.t, sink_count=len(head.sink), counts=head.counts(),
                                xi=head.xis()))
            meta.append(row)
        return dict(origin=origin, mu=mu, pe=pe, k=kr, v=vv, meta=meta)

    def select_margins(self, layer: int | None = None) -> np.ndarray:
        """Relative margins of every selection decision taken so far (the margin audit)."""
        layers = range(self.cfg.num_layers) if layer is None else [layer]
        out = []
        for l in layers:
            for row in self.heads[l]:
                for head in row:
                    out.extend(e.margin for e in head.events if e.kind in ("select_in", "select_keep"))
        return np.asarray(out, dtype=np.float64)
