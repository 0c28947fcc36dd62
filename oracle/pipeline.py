"""The DF-P2S per-frame steps in plain fp64 numpy (test infrastructure).

Step 1: N unit-variance fields with auto-covariance A_jj by FFT
  sampling, then point-wise Noll mixing a = L f (Eq.10).
  Noise (reading Q8): Hermitian spectral white noise per mode, two modes per
  complex inverse DFT: Y_p = sqrt(S_a) eta_a + i sqrt(S_b) eta_b, y = IDFT(Y),
  f_a = Re y, f_b = Im y.  eta is drawn with Philox4x32-10 (oracle/philox.py):
  for the canonical bin of each +-k pair eta = sqrt(PQ/2)(g1 + i g2), its mirror
  gets the conjugate, self-conjugate bins eta = sqrt(PQ) g1.
  Temporal AR(1) option (reading Q18): eta_t = alpha eta_{t-1} +
  sqrt(1 - alpha^2) xi_t, eta_0 = xi_0.
Step 2 (reading Q12): tilt warp Iw(x) = I(x + kappa (a_2, a_3)), bilinear,
  clamp-to-edge.
Step 3 (reading Q13): w = W3 ReLU(W2 ReLU(W1 a_{4..N} + b1) + b2) + b3.
Step 4 (Eq.9; readings Q14/Q15): out_c(x) = sum_k w_k(x) (h_k (*) Iw_c)(x),
  true convolution, centre tap T//2, whole-sample mirror boundary.
Step 5 (reading Q16): optional PSF-sum normalisation, additive Gaussian noise
  (Philox stream 1), clamp to [0, 1].
"""
from __future__ import annotations

import numpy as np

from .philox import STREAM_FIELD, STREAM_OUTPUT_NOISE, gaussians

N_MODES = 36


def n_pairs(N: int = N_MODES) -> int:
    return (N - 1 + 1) // 2  # modes 2..N, two per complex transform


def bin_symmetry(P: int, Q: int):
    """(canonical index, is_canonical, is_self_conjugate) for every bin (ky, kx)."""
    ky, kx = np.meshgrid(np.arange(P), np.arange(Q), indexing="ij")
    lin = ky * Q + kx
    lin_m = ((P - ky) % P) * Q + (Q - kx) % Q
    canon = np.minimum(lin, lin_m)
    return canon, lin == canon, lin == lin_m


def eta_from_gaussians(g1: np.ndarray, g2: np.ndarray) -> np.ndarray:
    """Hermitian spectral noise from per-bin Gaussians evaluated at the canonical bin.

    g1, g2 are [P][Q] arrays already indexed by each bin's canonical index.
    eta = sqrt(PQ/2)(g1 + i g2) on canonical bins, the conjugate on their mirrors,
    sqrt(PQ) g1 on self-conjugate bins, so E[eta_k conj(eta_k')] = PQ delta_kk'.
    """
    P, Q = g1.shape
    _, is_canon, is_self = bin_symmetry(P, Q)
    z = np.sqrt(P * Q / 2.0) * (g1 + 1j * np.where(is_canon, g2, -g2))
    return np.where(is_self, np.sqrt(P * Q) * g1 + 0j, z)


def white_spectral_noise(seed: int, frame: int, P: int, Q: int, N: int = N_MODES) -> np.ndarray:
    """xi_t: Hermitian complex white noise per mode slot (j = 2..N), [N-1][P][Q] complex128.

    Pair p (modes j = 2p+2, 2p+3) uses Philox counter (canonical bin, p | 0 << 16,
    frame) -- words (x0, x1) for mode a, (x2, x3) for mode b.
    """
    canon, _, _ = bin_symmetry(P, Q)
    eta = np.empty((N - 1, P, Q), dtype=np.complex128)
    for p in range(n_pairs(N)):
        (ga1, ga2), (gb1, gb2) = gaussians(canon, p, STREAM_FIELD, frame, seed)
        eta[2 * p] = eta_from_gaussians(ga1, ga2)
        if 2 * p + 1 < N - 1:
            eta[2 * p + 1] = eta_from_gaussians(gb1, gb2)
    return eta


def flow_phase_1d(n: int, s: float) -> np.ndarray:
    """Shift factor of one axis for a translation by s pixels (reading Q23): bin k gets
    exp(-2 pi i f_k s) with the signed frequency f_k = k/n (k < n/2), (k-n)/n (k > n/2);
    the Nyquist bin k = n/2 (its own mirror) gets the real cos(pi s), so the shifted
    spectrum stays Hermitian and the fields stay real.  For integer s this is exactly
    the periodic roll by s."""
    k = np.arange(n)
    ks = np.where(k <= n // 2, k, k - n).astype(np.float64)
    ph = np.exp(-2j * np.pi * ks * s / n)
    if n % 2 == 0:
        ph[n // 2] = np.cos(np.pi * s)
    return ph


def frozen_flow_noise(seed: int, t: int, P: int, Q: int, flow, N: int = N_MODES) -> np.ndarray:
    """Frozen flow: the coefficient fields of frame t are the frame-0 fields
    translated by t * (vx, vy) pixels, a(x, t) = a(x - v t, 0), on the periodic grid.  In
    the spectral domain that is the frame-0 noise times the per-axis shift factors."""
    vx, vy = flow
    eta = white_spectral_noise(seed, 0, P, Q, N)
    ph = np.outer(flow_phase_1d(P, vy * t), flow_phase_1d(Q, vx * t))
    return eta * ph[None]


def spectral_noise_sequence(seed: int, frame0: int, F: int, P: int, Q: int,
                            alpha: float = 0.0, N: int = N_MODES, flow=None):
    """eta_t for t = frame0 .. frame0+F-1 (AR(1) replayed from t = 0 if alpha != 0; frozen
    flow if flow = (vx, vy) px/frame is nonzero)."""
    if flow is not None and (flow[0] != 0.0 or flow[1] != 0.0):
        for t in range(frame0, frame0 + F):
            yield frozen_flow_noise(seed, t, P, Q, flow, N)
        return
    if alpha == 0.0:
        for t in range(frame0, frame0 + F):
            yield white_spectral_noise(seed, t, P, Q, N)
        return
    c = np.sqrt(1.0 - alpha * alpha)
    eta = None
    for t in range(0, frame0 + F):
        xi = white_spectral_noise(seed, t, P, Q, N)
        eta = xi if t == 0 else alpha * eta + c * xi
        if t >= frame0:
            yield eta


def fields_from_noise(eta: np.ndarray, sqrtS: np.ndarray, H: int, W: int) -> np.ndarray:
    """f[slot] (j = slot+2) = Re/Im of IDFT(sqrt(S_a) eta_a + i sqrt(S_b) eta_b), cropped."""
    M = eta.shape[0]
    f = np.empty((M, H, W))
    for p in range((M + 1) // 2):
        a, b = 2 * p, 2 * p + 1
        Y = sqrtS[a] * eta[a]
        if b < M:
            Y = Y + 1j * sqrtS[b] * eta[b]
        y = np.fft.ifft2(Y)  # (1/PQ) sum_k Y[k] e^{+2 pi i k.x}
        f[a] = y.real[:H, :W]
        if b < M:
            f[b] = y.imag[:H, :W]
    return f


def mix(f: np.ndarray, L: np.ndarray) -> np.ndarray:
    """a(x) = L f(x) per pixel (Eq.10); a_1 (piston) = 0.  f is slots j=2..N."""
    N = L.shape[0]
    a = np.zeros((N,) + f.shape[1:])
    a[1:] = np.einsum("ij,jhw->ihw", L[1:, 1:], f)
    return a


def sample_zernike(seed, frame0, F, sqrtS, L, H, W, alpha=0.0, flow=None):
    """a [F][N][H][W] for frames frame0 .. frame0+F-1 (step 1)."""
    P, Q = sqrtS.shape[-2:]
    N = L.shape[0]
    out = np.empty((F, N, H, W))
    for i, eta in enumerate(spectral_noise_sequence(seed, frame0, F, P, Q, alpha, N, flow)):
        out[i] = mix(fields_from_noise(eta, sqrtS, H, W), L)
    return out


def warp(img: np.ndarray, a2: np.ndarray, a3: np.ndarray, kappa: float) -> np.ndarray:
    """Iw_c(y, x) = bilinear(I_c, x + kappa a2, y + kappa a3), clamp-to-edge (step 2)."""
    C, H, W = img.shape
    yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    X = xx + kappa * a2
    Y = yy + kappa * a3
    x0 = np.floor(X)
    y0 = np.floor(Y)
    tx, ty = X - x0, Y - y0
    x0i = x0.astype(np.int64)
    y0i = y0.astype(np.int64)
    xa, xb = np.clip(x0i, 0, W - 1), np.clip(x0i + 1, 0, W - 1)
    ya, yb = np.clip(y0i, 0, H - 1), np.clip(y0i + 1, 0, H - 1)
    out = np.empty((C, H, W))
    for c in range(C):
        I = img[c].astype(np.float64)
        out[c] = ((1 - ty) * ((1 - tx) * I[ya, xa] + tx * I[ya, xb])
                  + ty * ((1 - tx) * I[yb, xa] + tx * I[yb, xb]))
    return out


def mlp(x: np.ndarray, layers) -> np.ndarray:
    """P2S network: x [n_in][...] -> w [K][...]; ReLU on hidden layers, linear output."""
    shp = x.shape[1:]
    h = x.reshape(x.shape[0], -1)
    for li, (Wm, b) in enumerate(layers):
        h = Wm @ h + b[:, None]
        if li < len(layers) - 1:
            h = np.maximum(h, 0.0)
    return h.reshape((h.shape[0],) + shp)


def reflect_index(i, n):
    """Whole-sample mirror: -i for i < 0, 2n-2-i for i >= n (valid for |overshoot| < n)."""
    i = np.asarray(i)
    i = np.where(i < 0, -i, i)
    return np.where(i >= n, 2 * n - 2 - i, i)


def blur(Iw: np.ndarray, w: np.ndarray, basis: np.ndarray) -> np.ndarray:
    """out_c(x) = sum_k w_k(x) sum_u h_k[u + T//2] Iw_c(refl(x - u)) (Eq.9)."""
    C, H, W = Iw.shape
    K, T, _ = basis.shape
    c = T // 2
    out = np.zeros((C, H, W))
    for ch in range(C):
        Ip = np.pad(Iw[ch].astype(np.float64), c, mode="reflect")
        conv = np.zeros((K, H, W))
        for ty in range(T):
            for tx in range(T):
                sl = Ip[2 * c - ty:2 * c - ty + H, 2 * c - tx:2 * c - tx + W]
                conv += basis[:, ty, tx, None, None].astype(np.float64) * sl[None]
        out[ch] = np.einsum("khw,khw->hw", w, conv)
    return out


def blur_at(Iw: np.ndarray, w_at: np.ndarray, basis: np.ndarray, ys, xs) -> np.ndarray:
    """Eq.9 at sample pixels (ys[i], xs[i]); w_at [n][K].  Returns [C][n]."""
    C, H, W = Iw.shape
    K, T, _ = basis.shape
    c = T // 2
    ys = np.asarray(ys)
    xs = np.asarray(xs)
    u = np.arange(T) - c
    py = reflect_index(ys[:, None] - u[None, :], H)  # [n][T] rows for tap ty
    px = reflect_index(xs[:, None] - u[None, :], W)
    out = np.empty((C, ys.size))
    hb = basis.astype(np.float64)
    for ch in range(C):
        patch = Iw[ch][py[:, :, None], px[:, None, :]].astype(np.float64)  # [n][T][T]
        conv = np.einsum("ktu,ntu->nk", hb, patch)
        out[ch] = np.einsum("nk,nk->n", w_at, conv)
    return out


def step5(out, w, basis, seed, frame, sigma=0.0, normalize=False, clamp01=False):
    """Step 5 (reading Q16): out / g (g = sum_k w_k sum_u h_k) ; + sigma xi ; clamp [0,1]."""
    out = np.array(out, dtype=np.float64)
    C, H, W = out.shape
    if normalize:
        g = np.einsum("khw,k->hw", w, basis.reshape(basis.shape[0], -1).astype(np.float64).sum(1))
        out = out / g[None]
    if sigma != 0.0:
        idx = np.arange(H * W).reshape(H, W)
        for ch in range(C):
            (g1, _), _ = gaussians(idx, ch, STREAM_OUTPUT_NOISE, frame, seed)
            out[ch] = out[ch] + sigma * g1
    if clamp01:
        out = np.clip(out, 0.0, 1.0)
    return out


def step5_at(out_at, w_at, basis, seed, frame, ys, xs, W, sigma=0.0, normalize=False, clamp01=False):
    """step5 evaluated at sample pixels only: out_at [C][n] (Eq.9 at (ys, xs)), w_at [n][K].
    Same arithmetic as step5 (reading Q16) with the pixel index y*W + x as noise counter."""
    out = np.array(out_at, dtype=np.float64)
    C = out.shape[0]
    if normalize:
        g = np.asarray(w_at, dtype=np.float64) @ basis.reshape(basis.shape[0], -1).astype(np.float64).sum(1)
        out = out / g[None]
    if sigma != 0.0:
        idx = np.asarray(ys) * W + np.asarray(xs)
        for ch in range(C):
            (g1, _), _ = gaussians(idx, ch, STREAM_OUTPUT_NOISE, frame, seed)
            out[ch] = out[ch] + sigma * g1
    if clamp01:
        out = np.clip(out, 0.0, 1.0)
    return out


def simulate(img, img_frame_stride_is_zero, seed, frame0, F, sqrtS, L, basis, layers, kappa,
             alpha=0.0, sigma=0.0, normalize=False, clamp01=False, return_intermediates=False):
    """Steps 1-5 for frames frame0 .. frame0+F-1.  img is [F|1][C][H][W]."""
    img = np.asarray(img)
    H, W = img.shape[-2:]
    P, Q = sqrtS.shape[-2:]
    N = L.shape[0]
    outs, inter = [], []
    for i, eta in enumerate(spectral_noise_sequence(seed, frame0, F, P, Q, alpha, N)):
        a = mix(fields_from_noise(eta, sqrtS, H, W), L)
        I = img[0] if img_frame_stride_is_zero else img[i]
        Iw = warp(I, a[1], a[2], kappa)
        w = mlp(a[3:], layers)
        o = blur(Iw, w, basis)
        o = step5(o, w, basis, seed, frame0 + i, sigma, normalize, clamp01)
        outs.append(o)
        if return_intermediates:
            inter.append(dict(a=a, Iw=Iw, w=w))
    out = np.stack(outs)
    return (out, inter) if return_intermediates else out
