"""ctypes binding of the C oracle (oracle/p2s_oracle.c, libp2s_oracle.so).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain argument marshalling: numpy
float64 arrays in, numpy float64 arrays out.  The library is built by
__graft_entry__.build() (make -C oracle).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libp2s_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built: make -C oracle")
        L = ctypes.CDLL(LIB)
        vp, i32, i64, u64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.p2so_philox.argtypes = [vp, vp, vp]
        L.p2so_white_noise.argtypes = [u64, i64, i32, i32, i32, vp]
        L.p2so_ar_update.argtypes = [vp, vp, ctypes.c_size_t, dbl]
        L.p2so_fields.argtypes = [vp, vp, i32, i32, i32, i32, i32, vp]
        L.p2so_mix.argtypes = [vp, vp, i32, ctypes.c_size_t, vp]
        L.p2so_warp.argtypes = [vp, vp, vp, dbl, i32, i32, i32, vp]
        L.p2so_mlp.argtypes = [vp, ctypes.c_size_t, i32, i32, i32, i32, vp, vp]
        L.p2so_blur.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, i64, vp]
        L.p2so_step5.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, i64, u64, i64, dbl, i32, i32]
        L.p2so_simulate_frame.argtypes = [vp, u64, i64, vp, i32, i32, vp, i32, i32, i32, i32, dbl, vp, i32, i32, vp,
                                          i32, i32, dbl, i32, i32, vp]
        L.p2so_simulate_frame.restype = i32
        L.p2so_threads.restype = i32
        _lib = L
    return _lib


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def threads():
    return lib().p2so_threads()


def philox(ctr, key):
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().p2so_philox(_p(c), _p(k), _p(out))
    return out


def white_noise(seed, frame, P, Q, N=36):
    out = np.empty((N - 1, P, Q), np.complex128)
    lib().p2so_white_noise(seed, frame, P, Q, N, _p(out))
    return out


def ar_update(eta, xi, alpha):
    eta = _c(eta, np.complex128).copy()
    xi = _c(xi, np.complex128)
    lib().p2so_ar_update(_p(eta), _p(xi), eta.size * 2, float(alpha))
    return eta


def fields(eta, sqrtS, H, W):
    eta = _c(eta, np.complex128)
    sq = _c(sqrtS)
    M, P, Q = sq.shape
    f = np.empty((M, H, W))
    lib().p2so_fields(_p(eta), _p(sq), P, Q, H, W, M + 1, _p(f))
    return f


def mix(f, L):
    f = _c(f)
    L = _c(L)
    N = L.shape[0]
    HW = f[0].size
    a = np.empty((N,) + f.shape[1:])
    lib().p2so_mix(_p(f), _p(L), N, HW, _p(a))
    return a


def warp(img, a2, a3, kappa):
    img = _c(img)
    C, H, W = img.shape
    out = np.empty_like(img)
    lib().p2so_warp(_p(img), _p(_c(a2)), _p(_c(a3)), float(kappa), C, H, W, _p(out))
    return out


def mlp(x, packed, K, hidden=(100, 100)):
    x = _c(x)
    n_in = x.shape[0]
    HW = x[0].size
    w = np.empty((K,) + x.shape[1:])
    lib().p2so_mlp(_p(x), HW, n_in, hidden[0], hidden[1], K, _p(_c(packed)), _p(w))
    return w


def blur(Iw, w, basis, ys=None, xs=None):
    Iw = _c(Iw)
    C, H, W = Iw.shape
    K, T, _ = basis.shape
    if ys is None:
        out = np.empty((C, H, W))
        lib().p2so_blur(_p(Iw), _p(_c(w)), _p(_c(basis)), C, H, W, K, T, None, None, -1, _p(out))
        return out
    ys = _c(ys, np.int32)
    xs = _c(xs, np.int32)
    out = np.empty((C, ys.size))
    lib().p2so_blur(_p(Iw), _p(_c(w)), _p(_c(basis)), C, H, W, K, T, _p(ys), _p(xs), ys.size, _p(out))
    return out


def step5(out, w, basis, seed, frame, sigma=0.0, normalize=False, clamp01=False):
    out = _c(out).copy()
    C, H, W = out.shape
    K, T, _ = basis.shape
    lib().p2so_step5(_p(out), _p(_c(w)), _p(_c(basis)), C, H, W, K, T, None, None, -1, seed, frame, float(sigma),
                     int(normalize), int(clamp01))
    return out


def simulate_frame(img, seed, frame, sqrtS, L, packed, basis, kappa, hidden=(100, 100), sigma=0.0, normalize=False,
                   clamp01=False):
    img = _c(img)
    C, H, W = img.shape
    sq = _c(sqrtS)
    M, P, Q = sq.shape
    K, T, _ = basis.shape
    out = np.empty((C, H, W))
    rc = lib().p2so_simulate_frame(_p(img), seed, frame, _p(sq), P, Q, _p(_c(L)), M + 1, C, H, W, float(kappa),
                                   _p(_c(packed)), hidden[0], hidden[1], _p(_c(basis)), K, T, float(sigma),
                                   int(normalize), int(clamp01), _p(out))
    if rc:
        raise MemoryError("p2so_simulate_frame: allocation failed")
    return out
