"""Eq. 4 token span and sparsity -- oracle, test infra only."""

from __future__ import annotations


def token_span(cache_size: int, num_cascades: int) -> int:
    """S~ = (|C| / N) * sum_{i=1..N} 2**(i-1)   (Eq. 4)."""
    assert cache_size % num_cascades == 0
    return (cache_size // num_cascades) * sum(2 ** (i - 1) for i in range(1, num_cascades + 1))


def sparsity(cache_size: int, num_cascades: int, seq_len: int):
    """(overall, window) = (1 - |C|/S, 1 - |C|/S~)."""
    if seq_len < cache_size:
        raise ValueError("sparsity undefined for S < |C|")
    return 1.0 - cache_size / seq_len, 1.0 - cache_size / token_span(cache_size, num_cascades)


def stride_chunks(S: int, stride: int):
    """Alg. 1 ``stride(inputs, stride_size)``: consecutive [start, end) ranges, last one ragged."""
    return [(a, min(a + stride, S)) for a in range(0, S, stride)]
