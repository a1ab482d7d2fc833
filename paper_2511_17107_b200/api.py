"""Thin ctypes binding of libpcband.so (include/pcband.h).  Argument marshalling only: every step
of the operator, preconditioner and eigensolver runs in the library's CUDA kernels.

Device buffers are torch tensors (complex128, CUDA) of shape (ncols, 3 N^3) -- column-major
blocks with ld = tensor.stride(0).  Host arrays are numpy.  Any failure raises PcError; there is
no CPU fallback (the library must be built: ``make`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCBAND_LIB") or os.path.join(_HERE, "libpcband.so")  # override: tuning builds

PC_OK, PC_ENOTCONV = 0, 1
PC_EINVAL, PC_ENOTPD, PC_ECUDA, PC_ENOMEM, PC_ENUMERIC = -1, -2, -3, -4, -5
PC_EPS_DIAGONAL, PC_EPS_CROSSDOF, PC_EPS_TRIVIAL = 0, 1, 2
PC_SPACE_FOURIER, PC_SPACE_REAL = 0, 1
PC_FFT_TO_FOURIER, PC_FFT_TO_REAL = 0, 1
PC_HPD_ASSUMP1, PC_HPD_SDD, PC_HPD_ZERO_OFFD, PC_HPD_GUARANTEED = 1, 2, 4, 8
STAT_NAMES = ["fft_z_kah", "fft_mid", "eps", "fft_z_ka", "resid", "gram", "rr", "update", "other"]
EPS_MODES = {"diagonal": PC_EPS_DIAGONAL, "crossdof": PC_EPS_CROSSDOF, "trivial": PC_EPS_TRIVIAL}


class PcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libpcband error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libpcband.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise PcError(PC_EINVAL, f"{LIB_PATH} not built (run `make` or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, d, ll, ull = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong, ctypes.c_ulonglong
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    sig = {
        "pc_create": (i, [ctypes.POINTER(vp), dp, i, dp, ctypes.POINTER(ctypes.c_uint8), i, d, i]),
        "pc_apply": (i, [vp, dp, vp, vp, i, ll, i, vp]),
        "pc_precond": (i, [vp, dp, vp, vp, i, ll, vp]),
        "pc_apply_multi": (i, [vp, dp, i, ip, vp, vp, i, ll, vp]),
        "pc_precond_multi": (i, [vp, dp, i, ip, vp, vp, i, ll, vp]),
        "pc_apply_eps": (i, [vp, vp, vp, i, ll, vp]),
        "pc_fft3": (i, [vp, vp, vp, i, ll, i, vp]),
        "pc_bands": (i, [vp, dp, i, i, d, i, ull, dp, dp, ip, ip, vp]),
        "pc_gamma": (d, [vp, dp]),
        "pc_info": (i, [vp, ip, ctypes.POINTER(ctypes.c_size_t)]),
        "pc_set_option": (i, [vp, ctypes.c_char_p, d]),
        "pc_stats": (i, [vp, dp, i]),
        "pc_supported_n": (i, [ip, i]),
        "pc_debug_heevj": (i, [dp, i, dp, dp, ip]),
        "pc_debug_pass": (i, [vp, dp, i, i, i, vp, vp, vp, i, ll, d]),
        "pc_history": (i, [vp, dp, i, ip]),
        "pc_bench_block": (i, [vp, i, i, i, i, i, dp]),
        "pc_destroy": (None, [vp]),
        "pc_trim": (None, [i]),
        "pc_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc, allow=(PC_OK,)):
    if rc not in allow:
        raise PcError(rc, lib().pc_last_error().decode())
    return rc


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _stream_ptr(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _block(t, ctx=None):
    """(pointer, ncols, ld) of a torch complex128 CUDA block (ncols, >= 3N^3): contiguous columns, column
    stride >= column length (no expanded/overlapping views), and, given ctx, columns of >= 3N^3."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.complex128):
        raise PcError(PC_EINVAL, "device blocks must be CUDA complex128 torch tensors")
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.dim() != 2 or t.stride(-1) != 1:
        raise PcError(PC_EINVAL, "a block is (ncols, len) with contiguous columns")
    nc = t.shape[0]
    ld = t.stride(0) if nc > 1 else t.shape[-1]
    if ld < t.shape[-1]:
        raise PcError(PC_EINVAL, "column stride smaller than the column length (expanded or overlapping view)")
    if ctx is not None and t.shape[-1] < ctx.len:
        raise PcError(PC_EINVAL, f"columns hold {t.shape[-1]} < 3 N^3 = {ctx.len} values")
    return ctypes.c_void_p(t.data_ptr()), nc, ld


def _pair(ctx, X, Y, same_ld=True):
    """Input/output blocks of one call: equal leading dimension (the ABI has one ld), output at least as
    many columns as the input."""
    px, nc, ld = _block(X, ctx)
    py, ncy, ldy = _block(Y, ctx)
    if ncy < nc:
        raise PcError(PC_EINVAL, f"output block has {ncy} < {nc} columns")
    if nc > 1 and ldy != ld:
        raise PcError(PC_EINVAL, "input and output blocks must share the leading dimension")
    return px, py, nc, ld


class Ctx:
    """Owns one pc_ctx (pc_destroy on close / garbage collection)."""

    def __init__(self, handle, n):
        self.h = handle
        self.n = n

    @property
    def len(self):
        return 3 * self.n ** 3

    def close(self):
        if self.h:
            lib().pc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pc_supported_n():
    L = lib()
    cnt = L.pc_supported_n(None, 0)
    arr = (ctypes.c_int * cnt)()
    L.pc_supported_n(arr, cnt)
    return list(arr)


def pc_create(A, n, eps1, masks, eps_mode="crossdof", gamma_override=0.0, device=0) -> Ctx:
    """A: 3x3 (columns a_1..a_3); eps1: 3x3 complex; masks: uint8 (4, n, n, n)."""
    L = lib()
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64).reshape(3, 3))
    e = np.asarray(eps1, dtype=np.complex128).reshape(3, 3)
    e18 = np.ascontiguousarray(np.stack([e.real, e.imag], axis=-1).reshape(18))
    m = np.ascontiguousarray(np.asarray(masks, dtype=np.uint8).reshape(4 * n ** 3))
    mode = EPS_MODES[eps_mode] if isinstance(eps_mode, str) else int(eps_mode)
    h = ctypes.c_void_p()
    _check(L.pc_create(ctypes.byref(h), _dptr(A), int(n), _dptr(e18),
                       m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), mode, float(gamma_override), int(device)))
    return Ctx(h, int(n))


def pc_apply(ctx: Ctx, k, X, Y, space=PC_SPACE_FOURIER, stream=None):
    kk = np.ascontiguousarray(np.asarray(k, dtype=np.float64).reshape(3))
    px, py, nc, ld = _pair(ctx, X, Y)
    _check(lib().pc_apply(ctx.h, _dptr(kk), px, py, nc, ld, int(space), _stream_ptr(stream)))


def pc_precond(ctx: Ctx, k, R, P, stream=None):
    kk = np.ascontiguousarray(np.asarray(k, dtype=np.float64).reshape(3))
    pr, pp, nc, ld = _pair(ctx, R, P)
    _check(lib().pc_precond(ctx.h, _dptr(kk), pr, pp, nc, ld, _stream_ptr(stream)))


def _multik(kpts, kcol, ncols):
    kk = np.ascontiguousarray(np.asarray(kpts, dtype=np.float64).reshape(-1, 3))
    kc = np.ascontiguousarray(np.asarray(kcol, dtype=np.int32).reshape(-1))
    if kc.size < ncols:
        raise PcError(PC_EINVAL, "kcol needs one k index per column")
    return kk, kc


def pc_apply_multi(ctx: Ctx, kpts, kcol, X, Y, stream=None):
    """Y[j] = Op(kpts[kcol[j]]) X[j] for every column j, one launch sequence for all k (Fourier space)."""
    px, py, nc, ld = _pair(ctx, X, Y)
    kk, kc = _multik(kpts, kcol, nc)
    _check(lib().pc_apply_multi(ctx.h, _dptr(kk), kk.shape[0], kc.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                px, py, nc, ld, _stream_ptr(stream)))


def pc_precond_multi(ctx: Ctx, kpts, kcol, R, P, stream=None):
    """P[j] = K_P(kpts[kcol[j]])^{-1} R[j] for every column j (Fourier space)."""
    pr, pp, nc, ld = _pair(ctx, R, P)
    kk, kc = _multik(kpts, kcol, nc)
    _check(lib().pc_precond_multi(ctx.h, _dptr(kk), kk.shape[0], kc.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                  pr, pp, nc, ld, _stream_ptr(stream)))


def pc_apply_eps(ctx: Ctx, E, Y, stream=None):
    pe, py, nc, ld = _pair(ctx, E, Y)
    _check(lib().pc_apply_eps(ctx.h, pe, py, nc, ld, _stream_ptr(stream)))


def pc_fft3(ctx: Ctx, X, Y, direction=PC_FFT_TO_FOURIER, stream=None):
    px, py, nc, ld = _pair(ctx, X, Y)
    _check(lib().pc_fft3(ctx.h, px, py, nc, ld, int(direction), _stream_ptr(stream)))


def pc_bands(ctx: Ctx, kpts, nev, tol=1e-5, maxit=500, seed=0, evecs=None, allow_notconv=True):
    """Returns dict(omega2 (nk, nev), resid (nk, nev), iters (nk,), status (nk,), rc)."""
    k = np.ascontiguousarray(np.asarray(kpts, dtype=np.float64).reshape(-1, 3))
    nk = k.shape[0]
    om = np.zeros((nk, nev))
    rs = np.zeros((nk, nev))
    it = np.zeros(nk, dtype=np.int32)
    stt = np.zeros(nk, dtype=np.int32)
    ev = None
    if evecs is not None:
        import torch
        need = nk * nev * ctx.len
        if not (isinstance(evecs, torch.Tensor) and evecs.is_cuda and evecs.dtype == torch.complex128
                and evecs.is_contiguous() and evecs.numel() >= need):
            raise PcError(PC_EINVAL, f"evecs must be a contiguous CUDA complex128 tensor of >= {need} elements")
        ev = ctypes.c_void_p(evecs.data_ptr())
    allow = (PC_OK, PC_ENOTCONV) if allow_notconv else (PC_OK,)
    rc = _check(lib().pc_bands(ctx.h, _dptr(k), nk, int(nev), float(tol), int(maxit), int(seed), _dptr(om), _dptr(rs),
                               it.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                               stt.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), ev), allow)
    return {"omega2": om, "resid": rs, "iters": it, "status": stt, "rc": rc}


def pc_gamma(ctx: Ctx, k):
    kk = np.ascontiguousarray(np.asarray(k, dtype=np.float64).reshape(3))
    return lib().pc_gamma(ctx.h, _dptr(kk))


def pc_info(ctx: Ctx):
    f = ctypes.c_int()
    w = ctypes.c_size_t()
    _check(lib().pc_info(ctx.h, ctypes.byref(f), ctypes.byref(w)))
    return {"hpd_flags": f.value, "ws_bytes_per_col": w.value}


def pc_set_option(ctx: Ctx, key: str, value: float):
    _check(lib().pc_set_option(ctx.h, key.encode(), float(value)))


def pc_stats(ctx: Ctx, reset=False):
    """Per kernel class: timed groups, CUDA-event ms, algorithmic flops and bytes; plus total launches."""
    out = np.zeros(4 * len(STAT_NAMES) + 1)
    _check(lib().pc_stats(ctx.h, _dptr(out), 1 if reset else 0))
    st = {nm: {"count": int(out[4 * i]), "ms": float(out[4 * i + 1]), "flops": float(out[4 * i + 2]),
               "bytes": float(out[4 * i + 3])} for i, nm in enumerate(STAT_NAMES)}
    st["launches"] = int(out[-1])
    return st


def pc_history(ctx: Ctx):
    """(iterations, b) array of Res_j for the last solved k-point."""
    b = ctypes.c_int()
    rows = lib().pc_history(ctx.h, None, 0, ctypes.byref(b))
    out = np.zeros(max(1, rows * b.value))
    lib().pc_history(ctx.h, _dptr(out), rows, ctypes.byref(b))
    return out[: rows * b.value].reshape(rows, b.value)


def pc_bench_block(ctx: Ctx, which: int, b: int, na: int, nP: int, reps: int = 10) -> float:
    """Mean milliseconds of one LOBPCG block-kernel launch group on random data (timing only)."""
    ms = ctypes.c_double()
    _check(lib().pc_bench_block(ctx.h, int(which), int(b), int(na), int(nP), int(reps), ctypes.byref(ms)))
    return ms.value


def pc_trim(device=-1):
    """Return cached device blocks of destroyed contexts to the driver (all devices by default)."""
    lib().pc_trim(int(device))


def pc_debug_pass(ctx: Ctx, k, kind, axis, direction, X, Y, XH=None, scale=1.0):
    """One FFT pass (test/tuning entry): kind 0 plain, 1 K_A^H-fused inverse z, 2 K_A + gamma K_B forward z
    (XH = the apply input x_hat).  Runs on the legacy default stream and synchronises."""
    kk = np.ascontiguousarray(np.asarray(k, dtype=np.float64).reshape(3))
    px, py, nc, ld = _pair(ctx, X, Y)
    pxh = _block(XH, ctx)[0] if XH is not None else None
    _check(lib().pc_debug_pass(ctx.h, _dptr(kk), int(kind), int(axis), int(direction), px, py, pxh, nc, ld,
                               float(scale)))


def pc_debug_heevj(A):
    A = np.asarray(A, dtype=np.complex128)
    n = A.shape[0]
    a = np.ascontiguousarray(A.T).view(np.float64).reshape(-1)  # column-major
    w = np.zeros(n)
    v = np.zeros(2 * n * n)
    sw = ctypes.c_int()
    _check(lib().pc_debug_heevj(_dptr(a), n, _dptr(w), _dptr(v), ctypes.byref(sw)))
    V = v.view(np.complex128).reshape(n, n).T.copy()
    return w, V, sw.value
