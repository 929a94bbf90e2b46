"""Alg. 2 (Cascading Sink Cache) with circular buffers -- oracle, test infra only.

Restates PAPER.md:588-626 (``alg:cascade``) line by line:

    if not sink.is_full():      sink U item; return
    for buf in cascade:
        if buf.is_accepting_tokens():
            if not buf.is_full(): buf U item; return
            else: buf U item; item <- buf.evict_oldest()
        else:
            if not buf.is_full(): buf U item; return   # eager add
            else:                                      # token selection
                if score(item) > score(newest): evict_newest; buf U item
                return
    (an item carried past the last sub-cache is dropped)

Circular buffers: each sub-cache keeps the slot of its oldest token xi;
insertion into a full buffer overwrites slot xi and xi <- (xi + 1) mod |C_i|.
"buf U item; item <- buf.evict_oldest()" on a full buffer is therefore the
overwrite of slot xi returning its previous occupant (reading Q19).

Readings used:
  Q1  acceptance counter: t = 0-based stream index of the token being offered,
      sink insertions included; sub-cache i (1-indexed) accepts iff
      t mod 2**(i-1) == 0  ("every 2nd ... every 4th iteration").
  Q2  strict '>' at selection: on a tie the resident stays.
  Q16 sinks are outside the |C| budget.
  Q14 |C| must be divisible by N (equal sub-caches).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple


@dataclass
class Token:
    """One cached token: origin = stream index, payload k/v (any object), mu = EMA score."""

    origin: int
    k: object = None
    v: object = None
    mu: float = 0.0


class Ring:
    """One sub-cache C_i as a circular buffer with oldest-slot pointer xi."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("sub-cache capacity must be >= 1")
        self.cap = capacity
        self.slots: List[Optional[Token]] = [None] * capacity
        self.xi = 0
        self.count = 0

    def is_full(self) -> bool:
        return self.count == self.cap

    def push(self, item: Token) -> Optional[Token]:
        """'buf U item' -- returns the evicted oldest token when the buffer was full."""
        if not self.is_full():
            # not full: occupied slots are exactly [0, count) and xi = count mod cap
            slot = self.count
            self.slots[slot] = item
            self.count += 1
            self.xi = self.count % self.cap
            return None
        slot = self.xi
        evicted = self.slots[slot]
        self.slots[slot] = item
        self.xi = (self.xi + 1) % self.cap          # xi^(t+1) = (xi^(t) + 1) mod |C_i|
        return evicted

    def newest_slot(self) -> int:
        """Slot of the most recently inserted token (the one before xi)."""
        assert self.count > 0
        return (self.xi - 1) % self.cap if self.is_full() else self.count - 1

    def newest(self) -> Token:
        return self.slots[self.newest_slot()]

    def replace_newest(self, item: Token) -> Token:
        """'evict_newest(); buf U item' on a full buffer: the newest slot gets item, xi unchanged."""
        s = self.newest_slot()
        old = self.slots[s]
        self.slots[s] = item
        return old

    def oldest_to_newest(self) -> List[Token]:
        if not self.is_full():
            return [self.slots[i] for i in range(self.count)]
        return [self.slots[(self.xi + j) % self.cap] for j in range(self.cap)]

    def slot_rank(self, slot: int) -> int:
        """Age rank of a slot within this buffer (0 = oldest)."""
        return (slot - self.xi) % self.cap if self.is_full() else slot


@dataclass
class Event:
    t: int
    kind: str           # sink | fill | eager | accept | select_in | select_keep | drop_end
    origin: int
    level: int          # 0 = sink, 1..N sub-cache
    margin: float = float("nan")   # relative margin |mu_a - mu_b| / max(mu_a, mu_b) for selects


class CascadeHead:
    """State of one (layer, sequence, kv-head) cascade: sink buffer + N rings + counter t."""

    def __init__(self, sink_size: int, cache_size: int, num_cascades: int,
                 selection: bool = True):
        if num_cascades < 1:
            raise ValueError("N >= 1")
        if cache_size % num_cascades != 0:             # Q14
            raise ValueError("|C| must be divisible by N")
        self.alpha = sink_size
        self.N = num_cascades
        self.c = cache_size // num_cascades
        self.sink: List[Token] = []
        self.rings = [Ring(self.c) for _ in range(num_cascades)]
        self.t = 0
        self.selection = selection
        self.events: List[Event] = []

    # ---- Alg. 2 -------------------------------------------------------------
    @staticmethod
    def accepting(level: int, t: int) -> bool:
        """Sub-cache `level` (1-indexed) accepts every 2**(level-1)-th iteration (Q1)."""
        return t % (1 << (level - 1)) == 0

    def add_token(self, item: Token) -> None:
        t = self.t
        self.t += 1
        if len(self.sink) < self.alpha:
            self.sink.append(item)
            self.events.append(Event(t, "sink", item.origin, 0))
            return
        for i, buf in enumerate(self.rings, start=1):
            if self.accepting(i, t):
                if not buf.is_full():
                    buf.push(item)
                    self.events.append(Event(t, "fill", item.origin, i))
                    return
                evicted = buf.push(item)
                self.events.append(Event(t, "accept", item.origin, i))
                item = evicted
            else:
                if not buf.is_full():                          # P:608-610 eager add
                    buf.push(item)
                    self.events.append(Event(t, "eager", item.origin, i))
                    return
                newest = buf.newest()                          # P:611-619 selection
                a, b = item.mu, newest.mu
                denom = max(a, b)
                margin = abs(a - b) / denom if denom > 0 else 0.0
                if self.selection and item.mu > newest.mu:     # strict '>' (Q2)
                    buf.replace_newest(item)
                    self.events.append(Event(t, "select_in", item.origin, i, margin))
                    self.events.append(Event(t, "drop_sel", newest.origin, i, margin))
                else:
                    self.events.append(Event(t, "select_keep", newest.origin, i, margin))
                    self.events.append(Event(t, "drop_sel", item.origin, i, margin))
                return
        self.events.append(Event(t, "drop_end", item.origin, self.N + 1))   # carried past C_N

    # ---- views ----------------------------------------------------------------
    def logical_order(self) -> List[Token]:
        """Residents ordered oldest -> newest: sinks, then C_N ... C_1 each oldest->newest.

        Every token in C_{i+1} is older than every token in C_i (tokens only move
        to deeper sub-caches), so this is ascending origin order."""
        out = list(self.sink)
        for buf in reversed(self.rings):
            out.extend(buf.oldest_to_newest())
        return out

    def n_resident(self) -> int:
        return len(self.sink) + sum(r.count for r in self.rings)

    def positions(self) -> List[Tuple[int, int]]:
        """(origin, pe) pairs: pe = rank of the token within the cache."""
        return [(tok.origin, pe) for pe, tok in enumerate(self.logical_order())]

    def counts(self) -> List[int]:
        return [r.count for r in self.rings]

    def xis(self) -> List[int]:
        return [r.xi for r in self.rings]


def reindex_positions(origins):
    """P:158 in isolation: tokens sorted by stream index receive pe = their index within the cache."""
    order = sorted(origins)
    return {o: i for i, o in enumerate(order)}
