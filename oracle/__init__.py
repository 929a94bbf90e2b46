"""CPU oracle for the Cascading KV Cache hot path (arXiv 2406.17808).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything in this package.  The product path (``paper_2406_17808_b200``) never
imports it, and this package never imports the product path: the two share
no code, headers, tables or constants.

Everything here is a plain, slow, obviously-correct restatement of the paper:

* ``cascade``    -- Alg. 2 with ring buffers,
                    step by step, plus the positional re-indexing of P:158.
* ``naive``      -- a second, independent model of Alg. 2 that keeps each
                    sub-cache as a shifting Python list (no xi pointer), used
                    only to cross-check ``cascade``.
* ``attention``  -- Eq. 1 / Eq. 2 attention with an exact fp64
                    softmax, rotary position encoding by cache rank,
                    and the per-key EMA-weighted probability mass of Alg. 3
                     in its exact-normaliser reading.
* ``model``      -- Alg. 1 strided prefill for a batch of
                    sequences and GQA head groups, with the EMA fold of
                    P:154 and the independent-head / max reduction of P:542.
* ``accounting`` -- Eq. 4 token span and the two sparsity formulas.

Floating point is float64 throughout (numpy).  Readings of the paper where it
is silent or ambiguous are listed in DESIGN.md section "Readings"; each
function cites the reading it uses (Q1..Q20).

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against values the paper prints, closed forms,
special cases or brute force.  The single unpinned convention is the phase of
the acceptance counter (reading Q1), which the paper does not fix; it is
frozen by the hand trace in ``tests/golden/toy_trace_alpha1_N2_c2.txt``.
"""
