"""Second, independent model of Alg. 2 -- oracle, test infra only.

Each sub-cache is a Python list kept oldest -> newest that *shifts* on eviction
(the concatenation-style cache the paper contrasts with).  There is no
xi pointer and no slot arithmetic, so a slot/xi bug in ``oracle.cascade`` cannot
be mirrored here.  Same readings Q1 (counter phase) and Q2 (strict '>').
"""

from __future__ import annotations

from typing import List


class NaiveCascade:
    def __init__(self, sink_size: int, cache_size: int, num_cascades: int,
                 selection: bool = True):
        assert cache_size % num_cascades == 0
        self.alpha = sink_size
        self.N = num_cascades
        self.c = cache_size // num_cascades
        self.sink: List[tuple] = []          # items are (origin, mu)
        self.levels: List[List[tuple]] = [[] for _ in range(num_cascades)]
        self.t = 0
        self.selection = selection
        self.dropped: List[int] = []

    def add(self, origin: int, mu: float = 0.0) -> None:
        t = self.t
        self.t += 1
        item = (origin, mu)
        if len(self.sink) < self.alpha:
            self.sink.append(item)
            return
        for idx, lst in enumerate(self.levels):
            period = 2 ** idx                      # level idx+1 accepts every 2**idx-th iteration
            full = len(lst) == self.c
            if t % period == 0:
                lst.append(item)
                if not full:
                    return
                item = lst.pop(0)                  # evict the oldest, carry it on
            else:
                if not full:
                    lst.append(item)
                    return
                if self.selection and item[1] > lst[-1][1]:
                    self.dropped.append(lst[-1][0])
                    lst[-1] = item
                else:
                    self.dropped.append(item[0])
                return
        self.dropped.append(item[0])

    def set_mu(self, fn) -> None:
        """Replace every resident's mu by fn(origin, mu)."""
        self.sink = [(o, fn(o, m)) for o, m in self.sink]
        self.levels = [[(o, fn(o, m)) for o, m in lst] for lst in self.levels]

    def logical_origins(self) -> List[int]:
        out = [o for o, _ in self.sink]
        for lst in reversed(self.levels):
            out.extend(o for o, _ in lst)
        return out

    def counts(self) -> List[int]:
        return [len(lst) for lst in self.levels]
