"""B200 (sm_100a) Cascading KV Cache hot path (arXiv 2406.17808): a C-ABI library
(`libcascade.so`, include/cascade.h) with a thin ctypes binding.

    from paper_2406_17808_b200 import Cascade, CascadeConfig, Stack

Importing the package does not load the library; the first Cascade / Stack does (and raises if it
has not been built: `python -m paper_2406_17808_b200.build`).  There is no CPU fallback."""


def __getattr__(name):
    # lazy: `import paper_2406_17808_b200.synth` (input generation) must not need the library
    if name in ("Cascade", "CascadeConfig", "CascadeError", "Stack"):
        from . import cascade
        return getattr(cascade, name)
    raise AttributeError(name)
