"""Thin ctypes binding of libcascade.so (include/cascade.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; PyTorch only provides
device memory (the workspace and I/O tensors) and streams.  There is no CPU fallback:
if the shared library is missing this module raises on import of the library.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# CASCADE_LIB selects an experiment build of the same sources (scripts/ A/B runs); default in-tree
LIB_PATH = os.environ.get("CASCADE_LIB", os.path.join(HERE, "libcascade.so"))

MAX_LEVELS = 16
F32, BF16 = 0, 1
OPT_ONEPASS_SCORES, OPT_EXACT_DECODE_ROPE = 1, 2
_STATUS = {0: "ok", -1: "invalid argument", -2: "invalid config", -3: "bad shape",
           -4: "call out of order", -5: "workspace", -6: "CUDA error", -7: "unsupported",
           -8: "handle poisoned by an earlier CUDA error"}


class CascadeError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {_STATUS.get(code, code)} ({code})")
        self.code = code


class _Config(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("sink_size", ctypes.c_int32),
                ("cache_size", ctypes.c_int32), ("num_cascades", ctypes.c_int32),
                ("max_stride", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("ema_gamma", ctypes.c_double), ("rope_theta", ctypes.c_double),
                ("softmax_scale", ctypes.c_double), ("head_policy", ctypes.c_int32),
                ("head_reduce", ctypes.c_int32), ("selection", ctypes.c_int32),
                ("options", ctypes.c_int32)]


class Mirror(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("sink_count", ctypes.c_int32),
                ("counts", ctypes.c_int32 * MAX_LEVELS), ("xi", ctypes.c_int32 * MAX_LEVELS)]


class _StateView(ctypes.Structure):
    _fields_ = [("mirror", Mirror), ("num_cascades", ctypes.c_int32),
                ("sub_cache_size", ctypes.c_int32), ("sink_size", ctypes.c_int32),
                ("slots_total", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("n_cached", ctypes.c_int32),
                ("k_raw", ctypes.c_void_p), ("v", ctypes.c_void_p), ("mu", ctypes.c_void_p),
                ("origin", ctypes.c_void_p), ("pe", ctypes.c_void_p)]


class _LayerWeights(ctypes.Structure):
    _fields_ = [("w_q", ctypes.c_void_p), ("w_k", ctypes.c_void_p), ("w_v", ctypes.c_void_p),
                ("w_o", ctypes.c_void_p)]


class _StackView(ctypes.Structure):
    _fields_ = [("m_last", ctypes.c_int32), ("x_in", ctypes.c_void_p), ("q", ctypes.c_void_p),
                ("k", ctypes.c_void_p), ("v", ctypes.c_void_p), ("o", ctypes.c_void_p),
                ("x_out", ctypes.c_void_p)]


_lib = None


def lib():
    """Loads libcascade.so once; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2406_17808_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, cfgp = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(_Config)
        sig = {
            "cascade_status_string": (ctypes.c_char_p, [i32]),
            "cascade_validate_config": (i32, [cfgp]),
            "cascade_workspace_bytes": (ctypes.c_size_t, [cfgp]),
            "cascade_init": (i32, [cfgp, vp, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(vp)]),
            "cascade_destroy": (None, [vp]),
            "cascade_prefill_stride": (i32, [vp, i32, vp, vp, vp, i32, vp, vp]),
            "cascade_prefill_stride_host": (i32, [vp, i32, vp, vp, vp, i32, vp, vp]),
            "cascade_prefill_stride_host_async": (i32, [vp, i32, vp, vp, vp, i32, vp, vp]),
            "cascade_host_wait": (i32, [vp]),
            "cascade_decode": (i32, [vp, i32, vp, vp, vp, vp, vp]),
            "cascade_state": (i32, [vp, i32, ctypes.POINTER(_StateView), vp]),
            "cascade_update_with_scores": (i32, [vp, i32, vp, vp, i32, vp, vp]),
            "cascade_last_scores": (i32, [vp, i32, vp, ctypes.POINTER(i32), vp]),
            "cascade_mirror_advance": (i32, [cfgp, ctypes.POINTER(Mirror), i32, vp, vp]),
            "cascade_launch_count": (ctypes.c_int64, [vp]),
            "cascade_reset": (i32, [vp, i32, vp]),
            "cascade_profile_enable": (i32, [vp, i32]),
            "cascade_profile_read": (i32, [vp, vp, vp, vp]),
            "cascade_attend": (i32, [vp, i32, vp, vp, vp, i32, vp, vp]),
            "cascade_score_buffer": (i32, [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(i32)]),
            "cascade_commit": (i32, [vp, i32, vp, vp, vp]),
            "cascade_load_state": (i32, [vp, i32, ctypes.POINTER(_StateView), vp]),
            "cascade_get_config": (i32, [vp, cfgp]),
            "cascade_stack_workspace_bytes": (ctypes.c_size_t, [cfgp, i32]),
            "cascade_stack_init": (i32, [vp, i32, ctypes.POINTER(_LayerWeights), vp, ctypes.c_size_t,
                                         ctypes.POINTER(vp)]),
            "cascade_stack_destroy": (None, [vp]),
            "cascade_stack_prefill": (i32, [vp, vp, ctypes.c_int64, i32, vp, vp]),
            "cascade_stack_trace": (i32, [vp, i32, ctypes.POINTER(_StackView)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


EXPORTED = ["cascade_status_string", "cascade_validate_config", "cascade_workspace_bytes",
            "cascade_init", "cascade_destroy", "cascade_prefill_stride",
            "cascade_prefill_stride_host", "cascade_prefill_stride_host_async", "cascade_host_wait",
            "cascade_decode", "cascade_state",
            "cascade_update_with_scores", "cascade_last_scores", "cascade_mirror_advance",
            "cascade_launch_count", "cascade_reset", "cascade_profile_enable",
            "cascade_profile_read", "cascade_attend", "cascade_score_buffer", "cascade_commit",
            "cascade_load_state", "cascade_get_config", "cascade_stack_workspace_bytes", "cascade_stack_init",
            "cascade_stack_destroy", "cascade_stack_prefill", "cascade_stack_trace"]


@dataclass
class CascadeConfig:
    num_layers: int = 1
    batch: int = 1
    num_q_heads: int = 32
    num_kv_heads: int = 8
    head_dim: int = 128
    sink_size: int = 64
    cache_size: int = 4096
    num_cascades: int = 4
    max_stride: int = 1024
    dtype: str = "bf16"
    ema_gamma: float = 0.9999
    rope_theta: float = 500000.0
    softmax_scale: float = 0.0
    head_reduce: str = "max"      # "max"; ablations "mean", "median"
    selection: bool = True        # False: the ablation without token selection (Q3)
    head_policy: str = "independent"   # or "homogeneous": one decision per sequence
    score_mode: str = "exact"     # or "onepass": the paper's one-pass estimator (Alg. 3)
    exact_decode_rope: bool = False   # decode key rotation with proven-exact bf16 rounding (Q17)

    def c_struct(self) -> _Config:
        return _Config(self.num_layers, self.batch, self.num_q_heads, self.num_kv_heads,
                       self.head_dim, self.sink_size, self.cache_size, self.num_cascades,
                       self.max_stride, BF16 if self.dtype == "bf16" else F32,
                       self.ema_gamma, self.rope_theta, self.softmax_scale,
                       {"independent": 0, "homogeneous": 1}[self.head_policy],
                       {"max": 0, "mean": 1, "median": 2}[self.head_reduce], int(self.selection),
                       {"exact": 0, "onepass": OPT_ONEPASS_SCORES}[self.score_mode] |
                       (OPT_EXACT_DECODE_ROPE if self.exact_decode_rope else 0))

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32

    @property
    def c(self) -> int:
        return self.cache_size // self.num_cascades

    @property
    def s_tot(self) -> int:
        return self.sink_size + self.cache_size


def _check(rc: int, where: str) -> None:
    if rc != 0:
        raise CascadeError(rc, where)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class _DevArray:
    """Exposes a device pointer to torch through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 2, "strides": None}


def workspace_bytes(cfg: CascadeConfig) -> int:
    return int(lib().cascade_workspace_bytes(ctypes.byref(cfg.c_struct())))


def validate(cfg: CascadeConfig) -> int:
    return int(lib().cascade_validate_config(ctypes.byref(cfg.c_struct())))


def mirror_advance(cfg: CascadeConfig, mirror: Mirror, m: int, want_pe=True, want_ops=True):
    """Host-only mirror advance (no GPU): returns (pe [S_tot] list or None, ops [4] list or None)."""
    import numpy as np
    pe = np.zeros(cfg.s_tot, dtype=np.int32) if want_pe else None
    ops = np.zeros(4, dtype=np.int64) if want_ops else None
    rc = lib().cascade_mirror_advance(ctypes.byref(cfg.c_struct()), ctypes.byref(mirror), m,
                                      None if pe is None else pe.ctypes.data_as(ctypes.c_void_p),
                                      None if ops is None else ops.ctypes.data_as(ctypes.c_void_p))
    _check(rc, "cascade_mirror_advance")
    return pe, ops


class Cascade:
    """One library handle: the cascades of every (layer, sequence, kv-head) on one device.

    The C ABI receives raw pointers and cannot check shapes, so every call checks here that
    each tensor has the shape, dtype, layout and device the handle's config implies (a wrong
    tensor would otherwise read or write out of bounds)."""

    def _check_io(self, ts, shapes, on_device=True, names=("q", "k", "v", "out")):
        for name, t, shape in zip(names, ts, shapes):
            if tuple(t.shape) != tuple(shape):
                raise ValueError(f"{name}: shape {tuple(t.shape)} != expected {tuple(shape)}")
            if t.dtype != self.cfg.torch_dtype or not t.is_contiguous():
                raise ValueError(f"{name}: needs a contiguous {self.cfg.torch_dtype} tensor")
            if on_device and t.device != self.device:
                raise ValueError(f"{name}: on {t.device}, the handle is on {self.device}")
            if not on_device and t.is_cuda:
                raise ValueError(f"{name}: the host-buffer call takes host tensors")

    def _chunk_shapes(self, m):
        c = self.cfg
        qs = (c.batch, m, c.num_q_heads, c.head_dim)
        ks = (c.batch, m, c.num_kv_heads, c.head_dim)
        return qs, ks, ks, qs

    def __init__(self, cfg: CascadeConfig, device: int = 0):
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        L = lib()
        cs = cfg.c_struct()
        rc = L.cascade_validate_config(ctypes.byref(cs))
        _check(rc, "cascade_validate_config")
        nbytes = int(L.cascade_workspace_bytes(ctypes.byref(cs)))
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self._h = ctypes.c_void_p()
        rc = L.cascade_init(ctypes.byref(cs), ctypes.c_void_p(base + off), nbytes, device,
                            ctypes.byref(self._h))
        _check(rc, "cascade_init")

    def close(self):
        if self._h:
            lib().cascade_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- hot path ------------------------------------------------------------
    def prefill_stride(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                       out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        m = q.shape[1]
        if out is None:
            out = torch.empty_like(q)
        self._check_io((q, k, v, out), self._chunk_shapes(m))
        rc = lib().cascade_prefill_stride(self._h, layer, _ptr(q), _ptr(k), _ptr(v), m, _ptr(out),
                                          _stream(stream))
        _check(rc, "cascade_prefill_stride")
        return out

    def prefill_stride_host(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                            out: torch.Tensor, stream=None) -> torch.Tensor:
        """q/k/v/out are (pinned) host tensors; copies happen inside the library call."""
        m = q.shape[1]
        self._check_io((q, k, v, out), self._chunk_shapes(m), on_device=False)
        rc = lib().cascade_prefill_stride_host(self._h, layer, _ptr(q), _ptr(k), _ptr(v), m,
                                               _ptr(out), _stream(stream))
        _check(rc, "cascade_prefill_stride_host")
        return out

    def prefill_stride_host_async(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                  out: torch.Tensor, stream=None) -> torch.Tensor:
        """Pipelined host-buffer step: returns at once; `out` is valid after host_wait()."""
        m = q.shape[1]
        self._check_io((q, k, v, out), self._chunk_shapes(m), on_device=False)
        rc = lib().cascade_prefill_stride_host_async(self._h, layer, _ptr(q), _ptr(k), _ptr(v), m,
                                                     _ptr(out), _stream(stream))
        _check(rc, "cascade_prefill_stride_host_async")
        return out

    def host_wait(self) -> None:
        _check(lib().cascade_host_wait(self._h), "cascade_host_wait")

    def decode(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
               out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(q)
        c = self.cfg
        qs, ks = (c.batch, c.num_q_heads, c.head_dim), (c.batch, c.num_kv_heads, c.head_dim)
        self._check_io((q, k, v, out), (qs, ks, ks, qs))
        rc = lib().cascade_decode(self._h, layer, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _stream(stream))
        _check(rc, "cascade_decode")
        return out

    # ---- split step (cross-device reduction of s between attention and update) ----
    def attend(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
               out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Attention + per-key mass of one step (cascade_attend); q/k/v shaped as for
        prefill_stride ([B, m, H, d]; m = 1 runs the fused decode kernel)."""
        m = q.shape[1]
        if out is None:
            out = torch.empty_like(q)
        self._check_io((q, k, v, out), self._chunk_shapes(m))
        rc = lib().cascade_attend(self._h, layer, _ptr(q), _ptr(k), _ptr(v), m, _ptr(out), _stream(stream))
        _check(rc, "cascade_attend")
        return out

    def score_buffer(self, layer: int) -> torch.Tensor:
        """The pending step's per-key mass [B, Hkv, S_tot + m] (a view of library memory: reduce
        it in place, e.g. dist.all_reduce(..., MAX), before commit)."""
        ptr, n = ctypes.c_void_p(), ctypes.c_int32(0)
        _check(lib().cascade_score_buffer(self._h, layer, ctypes.byref(ptr), ctypes.byref(n)),
               "cascade_score_buffer")
        shape = (self.cfg.batch, self.cfg.num_kv_heads, n.value)
        return torch.as_tensor(_DevArray(ptr.value, shape, "<f4"), device=self.device)

    def commit(self, layer: int, k: torch.Tensor, v: torch.Tensor, stream=None) -> None:
        _check(lib().cascade_commit(self._h, layer, _ptr(k), _ptr(v), _stream(stream)), "cascade_commit")

    def load_state(self, layer: int, st: dict, stream=None) -> None:
        """Restores a layer from a state dict as returned by state() (checkpoint restore)."""
        sv = _StateView()
        mr = sv.mirror
        mr.t, mr.sink_count = st["t"], st["sink_count"]
        for i, (cnt, xi) in enumerate(zip(st["counts"], st["xi"])):
            mr.counts[i], mr.xi[i] = cnt, xi
        sv.num_cascades, sv.sub_cache_size, sv.sink_size = self.cfg.num_cascades, self.cfg.c, self.cfg.sink_size
        sv.slots_total, sv.head_dim = self.cfg.s_tot, self.cfg.head_dim
        sv.dtype, sv.batch, sv.num_kv_heads = (BF16 if self.cfg.dtype == "bf16" else F32), self.cfg.batch, \
            self.cfg.num_kv_heads
        keep = [st[n].contiguous() for n in ("k", "v", "mu", "origin")]
        sv.k_raw, sv.v, sv.mu, sv.origin = (t.data_ptr() for t in keep)
        rc = lib().cascade_load_state(self._h, layer, ctypes.byref(sv), _stream(stream))
        (stream or torch.cuda.current_stream(self.device)).synchronize()   # `keep` is freed on return
        _check(rc, "cascade_load_state")

    # ---- test hooks / export ---------------------------------------------------
    def update_with_scores(self, layer: int, k: torch.Tensor, v: torch.Tensor, s: torch.Tensor,
                           stream=None) -> None:
        m = k.shape[1]
        _, ks, _, _ = self._chunk_shapes(m)
        self._check_io((k, v), (ks, ks), names=("k", "v"))
        if s.dtype != torch.float32 or s.device != self.device or not s.is_contiguous():
            raise ValueError("s: needs a contiguous float32 tensor on the handle's device")
        if tuple(s.shape) != (self.cfg.batch, self.cfg.num_kv_heads, self.cfg.s_tot + m):
            raise ValueError(f"s: shape {tuple(s.shape)}")
        rc = lib().cascade_update_with_scores(self._h, layer, _ptr(k), _ptr(v), m, _ptr(s),
                                              _stream(stream))
        _check(rc, "cascade_update_with_scores")

    def last_scores(self, layer: int, stream=None) -> torch.Tensor:
        m = ctypes.c_int32(0)
        # query m first with a dummy call that fails on size? -> keep a max-size buffer
        out = torch.empty((self.cfg.batch, self.cfg.num_kv_heads, self.cfg.s_tot + self.cfg.max_stride),
                          dtype=torch.float32, device=self.device)
        rc = lib().cascade_last_scores(self._h, layer, _ptr(out), ctypes.byref(m), _stream(stream))
        _check(rc, "cascade_last_scores")
        n = self.cfg.s_tot + m.value
        flat = out.view(-1)[: self.cfg.batch * self.cfg.num_kv_heads * n]
        return flat.view(self.cfg.batch, self.cfg.num_kv_heads, n).clone()

    def state(self, layer: int, stream=None) -> dict:
        """Copies of the layer's cascade state (torch tensors on the device) + the mirror."""
        sv = _StateView()
        rc = lib().cascade_state(self._h, layer, ctypes.byref(sv), _stream(stream))
        _check(rc, "cascade_state")
        B, Hk, S, d = self.cfg.batch, self.cfg.num_kv_heads, sv.slots_total, self.cfg.head_dim
        ts = "<f4" if self.cfg.dtype == "f32" else "<i2"

        def dev(ptr, shape, typestr, dtype=None):
            t = torch.as_tensor(_DevArray(ptr, shape, typestr), device=self.device).clone()
            return t.view(dtype) if dtype is not None else t

        kdt = torch.float32 if self.cfg.dtype == "f32" else torch.bfloat16
        mr = sv.mirror
        N = sv.num_cascades
        return dict(
            t=int(mr.t), sink_count=int(mr.sink_count), counts=[int(x) for x in mr.counts[:N]],
            xi=[int(x) for x in mr.xi[:N]], n_cached=int(sv.n_cached),
            k=dev(sv.k_raw, (B, Hk, S, d), ts, kdt), v=dev(sv.v, (B, Hk, S, d), ts, kdt),
            mu=dev(sv.mu, (B, Hk, S), "<f8"), origin=dev(sv.origin, (B, Hk, S), "<i8"),
            pe=dev(sv.pe, (S,), "<i4"))

    def launch_count(self) -> int:
        return int(lib().cascade_launch_count(self._h))

    def reset(self, layer: int, stream=None) -> None:
        _check(lib().cascade_reset(self._h, layer, _stream(stream)), "cascade_reset")

    def profile_enable(self, on: bool = True) -> None:
        _check(lib().cascade_profile_enable(self._h, 1 if on else 0), "cascade_profile_enable")

    PROFILE_CLASSES = ("prep", "attn_fwd", "attn_score", "maintenance", "decode_attn")

    def profile_read(self) -> dict:
        """{class: (ms_total, launch_groups, algorithmic_work)} since the last read."""
        import numpy as np
        ms = np.zeros(5, dtype=np.float64)
        cnt = np.zeros(5, dtype=np.int64)
        work = np.zeros(5, dtype=np.float64)
        _check(lib().cascade_profile_read(self._h, ms.ctypes.data_as(ctypes.c_void_p),
                                          cnt.ctypes.data_as(ctypes.c_void_p),
                                          work.ctypes.data_as(ctypes.c_void_p)), "cascade_profile_read")
        return {n: (float(ms[i]), int(cnt[i]), float(work[i])) for i, n in enumerate(self.PROFILE_CLASSES)}


class Stack:
    """A cascade_stack (include/cascade.h): Alg. 1's layer loop over the handle's L layers as
    synthetic attention layers (projections by cuBLASLt inside the library, attention and the cache
    update by the cascade kernels), driven as a wavefront over per-layer library streams.

    weights: L tuples (w_q [D, Hq d], w_k [D, Hkv d], w_v [D, Hkv d], w_o [Hq d, D]) of contiguous
    bf16 device tensors, kept alive by this object."""

    def __init__(self, cas: Cascade, weights, d_model: int):
        c = cas.cfg
        if c.dtype != "bf16":
            raise ValueError("the stack runs bf16 handles")
        if len(weights) != c.num_layers:
            raise ValueError("one weight set per layer")
        D, Hq, Hk, d = d_model, c.num_q_heads, c.num_kv_heads, c.head_dim
        shapes = ((D, Hq * d), (D, Hk * d), (D, Hk * d), (Hq * d, D))
        for l, ws in enumerate(weights):
            for name, t, shp in zip(("w_q", "w_k", "w_v", "w_o"), ws, shapes):
                if tuple(t.shape) != shp or t.dtype != torch.bfloat16 or not t.is_contiguous() \
                        or t.device != cas.device:
                    raise ValueError(f"layer {l} {name}: needs a contiguous bf16 {shp} tensor on {cas.device}")
        self.cas, self.D, self.weights = cas, D, [tuple(w) for w in weights]
        arr = (_LayerWeights * c.num_layers)(*[_LayerWeights(*(t.data_ptr() for t in ws)) for ws in self.weights])
        L = lib()
        nbytes = int(L.cascade_stack_workspace_bytes(ctypes.byref(c.c_struct()), D))
        if nbytes == 0:
            raise ValueError("invalid stack configuration")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=cas.device)
        base = self.workspace.data_ptr()
        self._s = ctypes.c_void_p()
        _check(L.cascade_stack_init(cas._h, D, arr, ctypes.c_void_p(base + (-base) % 256), nbytes,
                                    ctypes.byref(self._s)), "cascade_stack_init")

    def close(self):
        if self._s:
            lib().cascade_stack_destroy(self._s)
            self._s = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, x: torch.Tensor, m: int, y: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """x [B, T, D] bf16 (device, or pinned host) -> y [B, T, D] (same placement as given)."""
        c = self.cas.cfg
        if x.dim() != 3 or x.shape[0] != c.batch or x.shape[2] != self.D or x.dtype != torch.bfloat16 \
                or not x.is_contiguous():
            raise ValueError(f"x: needs a contiguous bf16 [{c.batch}, T, {self.D}] tensor")
        if y is None:
            y = torch.empty_like(x)
        if tuple(y.shape) != tuple(x.shape) or y.dtype != x.dtype or not y.is_contiguous():
            raise ValueError("y: needs x's shape and dtype")
        for name, t in (("x", x), ("y", y)):
            if t.is_cuda and t.device != self.cas.device:
                raise ValueError(f"{name}: on {t.device}, the stack is on {self.cas.device}")
            if not t.is_cuda and not t.is_pinned():
                raise ValueError(f"{name}: host tensors must be pinned")
        _check(lib().cascade_stack_prefill(self._s, _ptr(x), x.shape[1], m, _ptr(y), _stream(stream)),
               "cascade_stack_prefill")
        return y

    def trace(self, layer: int) -> dict:
        """The last chunk's intermediates of one layer (copies): x_in, q, k, v, o, x_out."""
        sv = _StackView()
        _check(lib().cascade_stack_trace(self._s, layer, ctypes.byref(sv)), "cascade_stack_trace")
        c, m = self.cas.cfg, sv.m_last
        B, Hq, Hk, d, D = c.batch, c.num_q_heads, c.num_kv_heads, c.head_dim, self.D
        shp = dict(x_in=(B, m, D), q=(B, m, Hq, d), k=(B, m, Hk, d), v=(B, m, Hk, d), o=(B, m, Hq, d),
                   x_out=(B, m, D))
        return {n: torch.as_tensor(_DevArray(getattr(sv, n), s, "<i2"), device=self.cas.device).clone()
                .view(torch.bfloat16) for n, s in shp.items()}
