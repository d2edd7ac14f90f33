"""Python binding of the LOVE C ABI (include/love.h).

Argument marshalling only: tensors are placed on the current CUDA device with the dtype the
ABI expects, pointers and the current stream are handed to liblove.so, results come back
as torch tensors.  Every step of the method runs in the library's CUDA kernels; if the
library or a GPU is missing this module raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _abi


class LoveError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_abi.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _lib():
    return _abi.load()


def _check(status: int) -> None:
    if status != _abi.LOVE_OK:
        msg = _lib().love_last_error()
        raise LoveError(status, msg.decode() if msg else "")


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dev(x, dtype: torch.dtype) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not x.is_cuda:
        x = x.to(device="cuda", dtype=dtype, non_blocking=True)
    elif x.dtype != dtype:
        x = x.to(dtype)
    return x.contiguous()


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _cache_fp64_mode(v) -> int:
    # love_opts.cache_fp64: "auto" (fp64 rebuild after an fp32 breakdown), True / "on", False / "off"
    if v is None or v == "auto":
        return _abi.LOVE_CACHE_FP64_AUTO
    if v is True or v == "on":
        return _abi.LOVE_CACHE_FP64_ON
    if v is False or v == "off":
        return _abi.LOVE_CACHE_FP64_OFF
    raise ValueError(f"cache_fp64: {v!r}")


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib().love_nccl_unique_id(buf))
    return buf.raw


def launch_count() -> int:
    return int(_lib().love_launch_count())


class LoveCache:
    """A built LOVE cache (Algorithm 1 pre-computation) on the current device."""

    def __init__(self, handle: int, precision: int, d: int, m_total: int, cache_precision: Optional[int] = None):
        self._h = ctypes.c_void_p(handle)
        self.precision = precision
        self.cache_precision = precision if cache_precision is None else cache_precision
        self.d = d
        self.m_total = m_total
        # outputs of predict_var / predict_covar / sample
        self.vdtype = torch.float64 if precision == _abi.LOVE_FP64 else torch.float32
        # the cache's factors (Rc, S exports) and the operator vectors (ski_mvm, kuu_mvm)
        self.cdtype = torch.float64 if self.cache_precision == _abi.LOVE_FP64 else torch.float32

    # ------------------------------------------------------------------ build
    @classmethod
    def build(cls, X, y, m: Sequence[int], lo: Sequence[float], h: Sequence[float],
              lengthscale: Sequence[float], outputscale: float, sigma2: float, k: int,
              precision: str = "fp32", prior: str = "ski", k_sample: int = 0, probe: str = "y",
              reorth_passes: int = 0, breakdown_tol: float = 0.0, lanczos_mode: str = "auto",
              var_blocks: str = "auto", reorth_tol: float = 0.0, cache_fp64="auto",
              rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
              stream=None) -> "LoveCache":
        d = len(m)
        Xd = _dev(X, torch.float64).reshape(-1, d)
        yd = _dev(y, torch.float64).reshape(-1)
        g = _abi.love_grid()
        g.d = d
        for i in range(d):
            g.m[i], g.lo[i], g.h[i] = int(m[i]), float(lo[i]), float(h[i])
        r = _abi.love_rbf()
        r.outputscale = float(outputscale)
        for i in range(d):
            r.lengthscale[i] = float(lengthscale[i])
        o = _abi.love_opts()
        o.precision = _abi.LOVE_FP64 if precision == "fp64" else _abi.LOVE_FP32
        o.probe = {"y": _abi.LOVE_PROBE_Y, "avg": _abi.LOVE_PROBE_AVGCOL}[probe]
        o.prior = _abi.LOVE_PRIOR_EXACT if prior == "exact" else _abi.LOVE_PRIOR_SKI
        o.reorth_passes = int(reorth_passes)
        o.breakdown_tol = float(breakdown_tol)
        o.k_sample = int(k_sample)
        o.lanczos_mode = {"auto": 0, "two_pass": 1, "one_read": 2, "partial": 3}[lanczos_mode]
        o.reorth_tol = float(reorth_tol)
        o.var_blocks = {"auto": 0, "off": 1}[var_blocks]
        o.cache_fp64 = _cache_fp64_mode(cache_fp64)
        dist = None
        idbuf = None
        if world > 1 or nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            dist = _abi.love_dist(rank, world, ctypes.cast(idbuf, ctypes.c_void_p))
        out = ctypes.c_void_p()
        _check(_lib().love_build_cache(ctypes.byref(g), ctypes.byref(r), float(sigma2), _ptr(Xd), _ptr(yd),
                                       int(Xd.shape[0]), int(k), ctypes.byref(o),
                                       ctypes.byref(dist) if dist is not None else None,
                                       ctypes.c_void_p(_stream(stream)), ctypes.byref(out)))
        return cls._made(out.value, o.precision, d, int(np.prod(m)))

    @classmethod
    def build_additive(cls, X, y, m: Sequence[int], lo: Sequence[float], h: Sequence[float],
                       lengthscale: Sequence[float], outputscale, sigma2: float, k: int,
                       precision: str = "fp32", prior: str = "ski", probe: str = "y",
                       reorth_passes: int = 0, breakdown_tol: float = 0.0, cache_fp64="auto",
                       rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                       stream=None) -> "LoveCache":
        """Additive composition of len(m) 1-D RBF components (Eq. 16);
        outputscale: one value for every component or one per component."""
        d = len(m)
        Xd = _dev(X, torch.float64).reshape(-1, d)
        yd = _dev(y, torch.float64).reshape(-1)
        s2 = list(outputscale) if hasattr(outputscale, "__len__") else [float(outputscale)] * d
        axes = (_abi.love_axis * d)()
        for e in range(d):
            axes[e].m, axes[e].lo, axes[e].h = int(m[e]), float(lo[e]), float(h[e])
            axes[e].lengthscale, axes[e].outputscale = float(lengthscale[e]), float(s2[e])
        o = _abi.love_opts()
        o.precision = _abi.LOVE_FP64 if precision == "fp64" else _abi.LOVE_FP32
        o.probe = {"y": _abi.LOVE_PROBE_Y, "avg": _abi.LOVE_PROBE_AVGCOL}[probe]
        o.prior = _abi.LOVE_PRIOR_EXACT if prior == "exact" else _abi.LOVE_PRIOR_SKI
        o.reorth_passes = int(reorth_passes)
        o.breakdown_tol = float(breakdown_tol)
        o.cache_fp64 = _cache_fp64_mode(cache_fp64)
        dist = None
        idbuf = None
        if world > 1 or nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            dist = _abi.love_dist(rank, world, ctypes.cast(idbuf, ctypes.c_void_p))
        out = ctypes.c_void_p()
        _check(_lib().love_build_cache_additive(axes, d, float(sigma2), _ptr(Xd), _ptr(yd), int(Xd.shape[0]),
                                                int(k), ctypes.byref(o),
                                                ctypes.byref(dist) if dist is not None else None,
                                                ctypes.c_void_p(_stream(stream)), ctypes.byref(out)))
        return cls._made(out.value, o.precision, d, int(sum(m)))

    @classmethod
    def _made(cls, handle: int, precision: int, d: int, m_total: int) -> "LoveCache":
        c = cls(handle, precision, d, m_total)
        inf = _abi.love_info()
        _check(_lib().love_cache_info(c._h, ctypes.byref(inf)))
        c.cache_precision = inf.cache_precision
        c.cdtype = torch.float64 if inf.cache_precision == _abi.LOVE_FP64 else torch.float32
        return c

    # ------------------------------------------------------------------ queries
    def predict_var(self, Xs, return_mean: bool = False, stream=None):
        Xd = _dev(Xs, torch.float64).reshape(-1, self.d)
        t = Xd.shape[0]
        var = torch.empty(t, dtype=self.vdtype, device=Xd.device)
        mean = torch.empty(t, dtype=self.vdtype, device=Xd.device) if return_mean else None
        _check(_lib().love_predict_var(self._h, _ptr(Xd), t, _ptr(var), _ptr(mean),
                                       ctypes.c_void_p(_stream(stream))))
        return (var, mean) if return_mean else var

    def predict_covar(self, Xa, Xb, stream=None):
        Xa = _dev(Xa, torch.float64).reshape(-1, self.d)
        Xb = _dev(Xb, torch.float64).reshape(-1, self.d)
        t = Xa.shape[0]
        out = torch.empty(t, dtype=self.vdtype, device=Xa.device)
        _check(_lib().love_predict_covar(self._h, _ptr(Xa), _ptr(Xb), t, _ptr(out),
                                         ctypes.c_void_p(_stream(stream))))
        return out

    def sample(self, Xs, s: int, seed: int = 0, zeta=None, stream=None):
        Xd = _dev(Xs, torch.float64).reshape(-1, self.d)
        t = Xd.shape[0]
        z = _dev(zeta, torch.float64) if zeta is not None else None
        out = torch.empty((s, t), dtype=self.vdtype, device=Xd.device)   # column-major t x s
        _check(_lib().love_sample(self._h, _ptr(Xd), t, int(s), int(seed),
                                  _ptr(z.t().contiguous() if z is not None else None),
                                  _ptr(out), ctypes.c_void_p(_stream(stream))))
        return out.t()

    # ------------------------------------------------------------------ operators
    def ski_mvm(self, v, stream=None):
        vd = _dev(v, self.cdtype)
        out = torch.empty_like(vd)
        _check(_lib().love_ski_mvm(self._h, _ptr(vd), _ptr(out), ctypes.c_void_p(_stream(stream))))
        return out

    def kuu_mvm(self, u, stream=None):
        ud = _dev(u, self.cdtype)
        out = torch.empty_like(ud)
        _check(_lib().love_kuu_mvm(self._h, _ptr(ud), _ptr(out), ctypes.c_void_p(_stream(stream))))
        return out

    # ------------------------------------------------------------------ introspection
    def info(self) -> dict:
        inf = _abi.love_info()
        _check(_lib().love_cache_info(self._h, ctypes.byref(inf)))
        k = inf.k_eff
        return dict(
            k_eff=k, k_pad=inf.k_pad, k_sample_eff=inf.k_sample_eff, n_local=inf.n_local,
            n_global=inf.n_global, m_total=inf.m_total, n_items=inf.n_items, b_norm=inf.b_norm,
            alpha=np.array([inf.alpha[i] for i in range(k)]),
            beta=np.array([inf.beta[i] for i in range(max(k - 1, 0))]),
            n_negative_var=inf.n_negative_var, n_out_of_range=inf.n_out_of_range,
            n_reorth_steps=inf.n_reorth_steps, precision=inf.precision, cache_precision=inf.cache_precision)

    def export(self, what: str, stream=None) -> torch.Tensor:
        code = {"rc": _abi.LOVE_EXPORT_RC, "mean": _abi.LOVE_EXPORT_MEAN, "S": _abi.LOVE_EXPORT_S,
                "perm": _abi.LOVE_EXPORT_PERM}[what]
        nb = ctypes.c_int64()
        _check(_lib().love_cache_export(self._h, code, None, 0, ctypes.byref(nb), None))
        dtype = {"rc": self.cdtype, "S": self.cdtype, "mean": torch.float64, "perm": torch.int32}[what]
        esize = torch.empty(0, dtype=dtype).element_size()
        out = torch.empty(nb.value // esize, dtype=dtype, device="cuda")
        _check(_lib().love_cache_export(self._h, code, _ptr(out), nb.value, None,
                                        ctypes.c_void_p(_stream(stream))))
        return out

    def free(self) -> None:
        if self._h is not None and self._h.value:
            _lib().love_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def build_cache(*args, **kwargs) -> LoveCache:
    return LoveCache.build(*args, **kwargs)
