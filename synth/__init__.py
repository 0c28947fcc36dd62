"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no Noll matrix, no PSD, no
FFT, no warp, no MLP evaluation, no blur).  It only draws the inputs that the
paper's workloads take from outside the simulator:

* ``image``       -- a clean image I_g (Eq.1 input), [C][H][W] float32 in [0,1]:
                     anisotropic Gaussian blobs + hard-edged rectangles + a
                     Siemens-star quadrant (stand-in for the paper's natural
                     images and monitor test patterns).
* ``basis``       -- a P2S spatial PSF basis phi_m (Eq.7) of K unit-sum
                     Gaussian blobs, [K][T][T] float32.
* ``mlp_weights`` -- random-init P2S network weights of the proposed shape
                     33 -> 100 -> 100 -> K, PyTorch
                     nn.Linear default init U(+-1/sqrt(fan_in)), packed
                     W1,b1,W2,b2,W3,b3 row-major [out][in].

All draws use numpy's Philox bit generator keyed by (seed, stream) so every
input is reproducible.  The per-frame noise that the *method* draws is NOT
produced here: the oracle and the CUDA path each implement Philox4x32-10
themselves.
"""
from __future__ import annotations

import numpy as np

# stream ids
STREAM_MLP = 2
STREAM_BASIS = 3
STREAM_IMAGE = 4


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), int(stream)]))


def image(H: int, W: int, C: int = 1, seed: int = 0) -> np.ndarray:
    """Synthetic clean image, float32 [C][H][W] in [0, 1]."""
    rng = _rng(seed, STREAM_IMAGE)
    yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    out = np.zeros((C, H, W), dtype=np.float64)
    for c in range(C):
        img = np.full((H, W), 0.15 + 0.1 * rng.random())
        # 48 anisotropic Gaussian blobs
        for _ in range(48):
            cy, cx = rng.random() * H, rng.random() * W
            sy = (0.01 + 0.08 * rng.random()) * H
            sx = (0.01 + 0.08 * rng.random()) * W
            th = rng.random() * np.pi
            amp = rng.uniform(-0.35, 0.6)
            dy, dx = yy - cy, xx - cx
            u = np.cos(th) * dx + np.sin(th) * dy
            v = -np.sin(th) * dx + np.cos(th) * dy
            img += amp * np.exp(-0.5 * ((u / sx) ** 2 + (v / sy) ** 2))
        # 16 hard-edged rectangles
        for _ in range(16):
            y0, x0 = int(rng.random() * H), int(rng.random() * W)
            h = max(1, int((0.03 + 0.2 * rng.random()) * H))
            w = max(1, int((0.03 + 0.2 * rng.random()) * W))
            img[y0:y0 + h, x0:x0 + w] = rng.random()
        # one Siemens-star quadrant in the lower-right corner
        r0 = 0.3 * min(H, W)
        dy, dx = yy - (H - 1), xx - (W - 1)
        rr = np.hypot(dy, dx)
        ang = np.arctan2(dy, dx)
        star = (np.sin(36.0 * ang) > 0).astype(np.float64)
        m = rr < r0
        img[m] = 0.05 + 0.9 * star[m]
        out[c] = img
    return np.clip(out, 0.0, 1.0).astype(np.float32)


def basis(K: int, T: int, seed: int = 0) -> np.ndarray:
    """K unit-sum Gaussian blobs on a T x T tap grid, float32 [K][T][T].

    sigma log-spaced in [0.6, T/6]; centre offsets uniform in +-1 px; a mild
    random anisotropy so the blobs are not separable.
    """
    if T % 2 != 1:
        raise ValueError("T must be odd")
    rng = _rng(seed, STREAM_BASIS)
    c = T // 2
    yy, xx = np.meshgrid(np.arange(T) - c, np.arange(T) - c, indexing="ij")
    sig = np.geomspace(0.6, T / 6.0, K) if K > 1 else np.array([0.6])
    out = np.zeros((K, T, T))
    for k in range(K):
        oy, ox = rng.uniform(-1, 1, size=2)
        a = sig[k] * rng.uniform(0.8, 1.25)
        b = sig[k] * rng.uniform(0.8, 1.25)
        th = rng.random() * np.pi
        dy, dx = yy - oy, xx - ox
        u = np.cos(th) * dx + np.sin(th) * dy
        v = -np.sin(th) * dx + np.cos(th) * dy
        g = np.exp(-0.5 * ((u / a) ** 2 + (v / b) ** 2))
        out[k] = g / g.sum()
    return out.astype(np.float32)


def mlp_sizes(n_in: int, hidden, K: int):
    dims = [n_in] + list(hidden) + [K]
    return [(dims[i + 1], dims[i]) for i in range(len(dims) - 1)]


def mlp_weights(K: int, hidden=(100, 100), n_in: int = 33, seed: int = 0) -> np.ndarray:
    """PyTorch nn.Linear default init, packed [W1(out,in), b1, W2, b2, W3, b3] float32."""
    rng = _rng(seed, STREAM_MLP)
    parts = []
    for (o, i) in mlp_sizes(n_in, hidden, K):
        bound = 1.0 / np.sqrt(i)
        parts.append(rng.uniform(-bound, bound, size=(o, i)).ravel())
        parts.append(rng.uniform(-bound, bound, size=(o,)))
    return np.concatenate(parts).astype(np.float32)


def unpack_mlp(packed: np.ndarray, K: int, hidden=(100, 100), n_in: int = 33):
    """Split a packed weight vector into [(W, b), ...] (float64 copies)."""
    packed = np.asarray(packed, dtype=np.float64)
    out, off = [], 0
    for (o, i) in mlp_sizes(n_in, hidden, K):
        W = packed[off:off + o * i].reshape(o, i)
        off += o * i
        b = packed[off:off + o]
        off += o
        out.append((W, b))
    if off != packed.size:
        raise ValueError(f"packed MLP has {packed.size} values, expected {off}")
    return out


# BASELINE.json configs: name -> dict
CONFIGS = {
    "cfg1_64": dict(H=64, W=64, C=1, F=1, d_over_r0=2.0, K=16, T=17, ar_alpha=0.0),
    "cfg2_256": dict(H=256, W=256, C=1, F=100, d_over_r0=3.0, K=100, T=33, ar_alpha=0.95),
    "cfg3_512": dict(H=512, W=512, C=3, F=64, d_over_r0=3.0, K=100, T=33, ar_alpha=0.0),
    "cfg4_1080p": dict(H=1080, W=1920, C=3, F=100, d_over_r0=4.0, K=100, T=33, ar_alpha=0.95),
    "cfg5_4k": dict(H=2160, W=3840, C=3, F=1, d_over_r0=5.0, K=100, T=33, ar_alpha=0.95),
}
NOISE_SEED = 2210
