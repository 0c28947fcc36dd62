"""Thin ctypes binding of include/p2s.h (argument marshalling only).

Every step of the simulator runs in libp2s.so (sm_100a CUDA kernels + host plan
code).  There is no Python or CPU fallback: if the library is missing or cannot be
loaded the import fails loudly.  torch is used only to hand over device pointers and
the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libp2s.so")

P2S_OK = 0
_STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "NUMERIC", 3: "CUDA", 4: "OUT_OF_MEMORY", 5: "UNSUPPORTED"}

# every entry point declared in include/p2s.h
EXPORTS = ("p2s_plan_create", "p2s_plan_destroy", "p2s_sample_zernike", "p2s_warp", "p2s_blur",
           "p2s_simulate_frames", "p2s_simulate_frames_host", "p2s_last_error", "p2s_plan_info",
           "p2s_plan_export_tables", "p2s_plan_import_sqrtS", "p2s_plan_stage_timing", "p2s_plan_stage_times", "p2s_field_autocorr", "p2s_exact_psf", "p2s_render_exact", "p2s_fit_basis", "p2s_fit_readout", "p2s_blur_weights", "p2s_correlation_energies", "p2s_aperture_stats", "p2s_train_mlp", "p2s_sample_zernike_from_noise",
           "p2s_philox_fill",
           "p2s_host_tables", "p2s_grid_size", "p2s_slab_geometry", "p2s_slab_counts", "p2s_slab_rows",
           "p2s_slab_finish")


class P2SError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"p2s error {status} ({_STATUS.get(status, '?')}): {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("taps", ctypes.c_int), ("aperture_m", ctypes.c_double), ("wavelength_m", ctypes.c_double),
                ("s_per_px", ctypes.c_double), ("tilt_px_per_rad", ctypes.c_double), ("pad", ctypes.c_int),
                ("mlp_hidden", ctypes.c_int * 2), ("max_batch", ctypes.c_int), ("ar_alpha", ctypes.c_float),
                ("noise_sigma", ctypes.c_float), ("normalize_psf_sum", ctypes.c_int), ("clamp01", ctypes.c_int),
                ("device", ctypes.c_int), ("flow_px_per_frame", ctypes.c_float * 2), ("slab_count", ctypes.c_int),
                ("slab_rank", ctypes.c_int), ("force", ctypes.c_uint)]


# p2s_options.force bits (include/p2s.h): kernel-selection overrides for tests / A-B runs
FORCE_FFT_GENERIC = 0x001
FORCE_FFT_SMALL_RADIX = 0x002
FORCE_AR_ROW_KERNEL = 0x004
FORCE_AR_PAIR_KERNEL = 0x008
FORCE_ROWS_PINGPONG = 0x010
FORCE_COLS_PER_BLOCK = 0x020
FORCE_X_PLANES = 0x040
FORCE_X_TILES = 0x080
FORCE_WARP_FUSION = 0x100
FORCE_BLUR_SINGLE = 0x200
FORCE_COLS_PERSISTENT = 0x400
FORCE_WARP_GATHER = 0x800
FORCE_X_OCTETS = 0x1000
FORCE_MLP_A1_THREADS = 0x2000


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (make -C paper_2210_06713_b200/csrc)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
    dp, fp = ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
    lib.p2s_plan_create.argtypes = [ctypes.POINTER(vp), i32, i32, i32, ctypes.c_double, ctypes.c_double, i32, i32,
                                    fp, fp, ctypes.POINTER(Options)]
    lib.p2s_plan_destroy.argtypes = [vp]
    lib.p2s_sample_zernike.argtypes = [vp, u64, i64, i32, vp, vp]
    lib.p2s_warp.argtypes = [vp, vp, i64, vp, vp, i32, vp]
    lib.p2s_blur.argtypes = [vp, vp, vp, u64, i64, vp, i32, vp]
    lib.p2s_simulate_frames.argtypes = [vp, vp, i64, u64, i64, i32, vp, vp]
    lib.p2s_simulate_frames_host.argtypes = [vp, vp, i64, u64, i64, i32, vp, vp]
    lib.p2s_last_error.restype = ctypes.c_char_p
    lib.p2s_plan_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_size_t), dp,
                                  ctypes.POINTER(i32)]
    lib.p2s_plan_export_tables.argtypes = [vp, vp, vp, vp]
    lib.p2s_plan_import_sqrtS.argtypes = [vp, vp]
    lib.p2s_plan_stage_timing.argtypes = [vp, i32]
    lib.p2s_plan_stage_times.argtypes = [vp, vp, vp]
    lib.p2s_philox_fill.argtypes = [u32, u32, u32, u32, u32, i64, vp, vp]
    lib.p2s_field_autocorr.argtypes = [vp, vp, i32, i32, vp, vp]
    lib.p2s_exact_psf.argtypes = [vp, vp, vp, i32, i32, vp, vp]
    lib.p2s_aperture_stats.argtypes = [vp, vp, i32, vp, i32, vp, vp]
    lib.p2s_fit_basis.argtypes = [vp, i32, i32, i32, vp, vp]
    lib.p2s_fit_readout.argtypes = [vp, i32, i32, i32, i32, vp, vp, i32, ctypes.c_double, vp, vp]
    lib.p2s_sample_zernike_from_noise.argtypes = [vp, vp, i32, vp, vp]
    lib.p2s_train_mlp.argtypes = [vp, i32, i32, i32, i32, vp, vp, i32, vp, i32, i32, ctypes.c_double, vp, vp]
    lib.p2s_correlation_energies.argtypes = [i32, ctypes.c_double, ctypes.c_double, i32, i32, i32, vp, vp, vp, vp]
    lib.p2s_blur_weights.argtypes = [vp, vp, vp, u64, i64, vp, i32, vp]
    lib.p2s_render_exact.argtypes = [vp, vp, vp, i32, vp, vp]
    lib.p2s_host_tables.argtypes = [i32, i32, ctypes.c_double, ctypes.c_double, i32, vp, vp, vp, vp]
    lib.p2s_slab_geometry.argtypes = [i32, i32, i32, i32, i32, i32, vp]
    lib.p2s_slab_counts.argtypes = [vp, vp, vp]
    lib.p2s_slab_rows.argtypes = [vp, u64, i64, vp, vp]
    lib.p2s_slab_finish.argtypes = [vp, vp, vp, u64, i64, vp, vp]
    lib.p2s_grid_size.argtypes = [i32]
    lib.p2s_grid_size.restype = i32
    for name in EXPORTS:
        if name not in ("p2s_last_error", "p2s_grid_size"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


lib = _load()


def _check(st):
    if st != P2S_OK:
        raise P2SError(st, lib.p2s_last_error().decode())


def _ptr(x):
    """Device pointer of a torch tensor (or an int address).  The C ABI takes dense
    row-major buffers, so a non-contiguous tensor is an error (never silently re-laid)."""
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if hasattr(x, "is_contiguous") and not x.is_contiguous():
        raise ValueError("p2s: tensor arguments must be contiguous (row-major); use .contiguous()")
    return ctypes.c_void_p(x.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def grid_size(x: int) -> int:
    return lib.p2s_grid_size(int(x))


SLAB_KEYS = ("x0", "x1", "hx0", "hx1", "kp0", "kp1", "rows", "P", "Q")


def slab_geometry(H, W, T, G, rank, pad=1):
    """Rank `rank`'s share of one H x W frame over G ranks (single-frame slab mode, NEXT-4):
    output columns [x0, x1), halo strip [hx0, hx1), Hermitian row pairs [kp0, kp1), rows."""
    info = np.zeros(9, dtype=np.int64)
    _check(lib.p2s_slab_geometry(H, W, T, pad, G, rank, info.ctypes.data))
    return dict(zip(SLAB_KEYS, (int(v) for v in info)))


def host_tables(P, Q, s_per_px, d_over_r0, Z=36, want_sqrtS=True):
    """Library plan-time tables computed on the host (no GPU): A0, L, sqrt(S), clamped fractions."""
    A0 = np.zeros((Z, Z))
    L = np.zeros((Z, Z))
    sq = np.zeros((Z - 1, P, Q)) if want_sqrtS else None
    cl = np.zeros(Z - 1) if want_sqrtS else None
    _check(lib.p2s_host_tables(P, Q, float(s_per_px), float(d_over_r0), Z, A0.ctypes.data, L.ctypes.data,
                               sq.ctypes.data if want_sqrtS else None, cl.ctypes.data if want_sqrtS else None))
    return A0, L, sq, cl


def fit_basis(psfs, M):
    """PCA basis of a PSF database (host float32 [n][T][T]) -> (basis [M+1][T][T], residual)."""
    psfs = np.ascontiguousarray(psfs, dtype=np.float32)
    n, T = psfs.shape[0], psfs.shape[1]
    basis = np.empty((M + 1, T, T), dtype=np.float32)
    res = ctypes.c_double()
    _check(lib.p2s_fit_basis(psfs.ctypes.data, n, T, M, basis.ctypes.data, ctypes.byref(res)))
    return basis, res.value


def fit_readout(mlp, a, beta, hidden=(100, 100), lam=1e-3):
    """Ridge fit of the MLP output layer: mlp (packed float32), a [n][n_in], beta [n][K] ->
    (packed float32 with fitted W3, b3, relative residual)."""
    mlp = np.ascontiguousarray(mlp, dtype=np.float32)
    a = np.ascontiguousarray(a, dtype=np.float32)
    beta = np.ascontiguousarray(beta, dtype=np.float32)
    out = np.empty_like(mlp)
    res = ctypes.c_double()
    _check(lib.p2s_fit_readout(mlp.ctypes.data, a.shape[1], hidden[0], hidden[1], beta.shape[1], a.ctypes.data,
                               beta.ctypes.data, a.shape[0], float(lam), out.ctypes.data, ctypes.byref(res)))
    return out, res.value


def correlation_energies(s_max, n_per_unit=24, Z=36, d_over_r0=1.0, angle_mean=True, mode_lo=4):
    """Approximation energies of P:369-397 -> (s, E, E~, E-), host float64 [ns+1]."""
    ns = max(2, int(round(n_per_unit * s_max)))
    out = [np.empty(ns + 1) for _ in range(4)]
    _check(lib.p2s_correlation_energies(Z, float(d_over_r0), float(s_max), n_per_unit, int(bool(angle_mean)),
                                        mode_lo, *[o.ctypes.data for o in out]))
    return tuple(out)


def train_mlp(mlp, a, beta, order, batch=256, lr=1e-3, hidden=(100, 100)):
    """Adam/MSE training of all MLP layers (reading Q26): mlp (packed float32), a [n][n_in],
    beta [n][K], order int32 [epochs][n] -> (trained packed float32, per-epoch loss)."""
    mlp = np.ascontiguousarray(mlp, dtype=np.float32)
    a = np.ascontiguousarray(a, dtype=np.float32)
    beta = np.ascontiguousarray(beta, dtype=np.float32)
    order = np.ascontiguousarray(order, dtype=np.int32)
    epochs = order.shape[0]
    out = np.empty_like(mlp)
    curve = np.empty(epochs)
    _check(lib.p2s_train_mlp(mlp.ctypes.data, a.shape[1], hidden[0], hidden[1], beta.shape[1], a.ctypes.data,
                             beta.ctypes.data, a.shape[0], order.ctypes.data, epochs, batch, float(lr),
                             out.ctypes.data, curve.ctypes.data))
    return out, curve


def philox_fill(c1, c2, c3, k0, k1, n, out, stream=None):
    _check(lib.p2s_philox_fill(c1, c2, c3, k0, k1, n, _ptr(out), _stream(stream)))


@dataclass
class PlanConfig:
    H: int
    W: int
    C: int
    d_over_r0: float
    L_m: float = 1000.0
    Z: int = 36
    K: int = 16
    taps: int = 17
    aperture_m: float = 0.0
    wavelength_m: float = 0.0
    s_per_px: float = 0.0
    tilt_px_per_rad: float = 0.0
    pad: int = 0
    mlp_hidden: tuple = (100, 100)
    max_batch: int = 0
    ar_alpha: float = 0.0
    noise_sigma: float = 0.0
    normalize_psf_sum: bool = False
    clamp01: bool = False
    device: int = 0
    flow: tuple = (0.0, 0.0)  # frozen flow (vx, vy) pixels per frame (NEXT-3)
    slab_count: int = 0  # >= 2: rank slab_rank's share of one frame (single-frame latency mode, NEXT-4)
    slab_rank: int = 0
    force: int = 0  # FORCE_* bits (kernel-selection overrides; 0 = production dispatch)
    extra: dict = field(default_factory=dict)


class Plan:
    """Owns a p2s_plan.  Buffers are torch CUDA tensors (float32, contiguous)."""

    def __init__(self, cfg: PlanConfig, basis: np.ndarray, mlp_weights: np.ndarray):
        self.cfg = cfg
        basis = np.ascontiguousarray(basis, dtype=np.float32)
        mlp = np.ascontiguousarray(mlp_weights, dtype=np.float32)
        o = Options()
        o.taps = cfg.taps
        o.aperture_m = cfg.aperture_m
        o.wavelength_m = cfg.wavelength_m
        o.s_per_px = cfg.s_per_px
        o.tilt_px_per_rad = cfg.tilt_px_per_rad
        o.pad = cfg.pad
        o.mlp_hidden[0], o.mlp_hidden[1] = cfg.mlp_hidden
        o.max_batch = cfg.max_batch
        o.ar_alpha = cfg.ar_alpha
        o.noise_sigma = cfg.noise_sigma
        o.normalize_psf_sum = int(cfg.normalize_psf_sum)
        o.clamp01 = int(cfg.clamp01)
        o.device = cfg.device
        o.flow_px_per_frame[0], o.flow_px_per_frame[1] = cfg.flow
        o.slab_count = cfg.slab_count
        o.slab_rank = cfg.slab_rank
        o.force = cfg.force
        self._h = ctypes.c_void_p()
        _check(lib.p2s_plan_create(ctypes.byref(self._h), cfg.H, cfg.W, cfg.C, float(cfg.d_over_r0),
                                   float(cfg.L_m), cfg.Z, cfg.K, basis.ctypes.data, mlp.ctypes.data, ctypes.byref(o)))
        P, Q, ws, cl, mb = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t(), ctypes.c_double(), ctypes.c_int()
        _check(lib.p2s_plan_info(self._h, ctypes.byref(P), ctypes.byref(Q), ctypes.byref(ws), ctypes.byref(cl),
                                 ctypes.byref(mb)))
        self.P, self.Q, self.workspace_bytes, self.clamped_psd_fraction, self.max_batch = \
            P.value, Q.value, ws.value, cl.value, mb.value

    def close(self):
        if self._h:
            lib.p2s_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- per-frame API
    def sample_zernike(self, seed, frame0, nframes, zern, stream=None):
        _check(lib.p2s_sample_zernike(self._h, seed, frame0, nframes, _ptr(zern), _stream(stream)))

    def field_autocorr(self, zern, nframes, max_lag, out, stream=None):
        """out (device float64 [Z][2][max_lag]) <- periodic auto-correlation of zern along x, y."""
        _check(lib.p2s_field_autocorr(self._h, _ptr(zern), nframes, max_lag, _ptr(out), _stream(stream)))

    def sample_zernike_from_noise(self, eta, nframes, zern, stream=None):
        """Step 1 from given spectral noise: eta device complex64 [F][Z-1][P][Q] -> zern."""
        _check(lib.p2s_sample_zernike_from_noise(self._h, _ptr(eta), nframes, _ptr(zern), _stream(stream)))

    def aperture_stats(self, zern, nframes, pixels, out, stream=None):
        """out (device float64 [3][32][63]) <- structure function, LE and SE OTF of the pupil
        phases of zern at the given pixels (device int32) over nframes frames."""
        _check(lib.p2s_aperture_stats(self._h, _ptr(zern), nframes, _ptr(pixels), pixels.numel(), _ptr(out),
                                      _stream(stream)))

    def blur_weights(self, warped, weights, seed, frame0, out, nframes, stream=None):
        """Steps 4-5 with given per-pixel basis weights (device float [F][K][H][W])."""
        _check(lib.p2s_blur_weights(self._h, _ptr(warped), _ptr(weights), seed, frame0, _ptr(out), nframes,
                                    _stream(stream)))

    def exact_psf(self, zern, pixels, n, include_tilt, out, stream=None):
        """out (device float [n][T][T]) <- Eq.2 PSFs of the given pixels of one frame."""
        _check(lib.p2s_exact_psf(self._h, _ptr(zern), _ptr(pixels), n, int(include_tilt), _ptr(out), _stream(stream)))

    def render_exact(self, img, zern, include_tilt, out, stream=None):
        """out (device float [C][H][W]) <- Eq.1 gather render of one frame with exact PSFs."""
        _check(lib.p2s_render_exact(self._h, _ptr(img), _ptr(zern), int(include_tilt), _ptr(out), _stream(stream)))

    def warp(self, img, img_frame_stride, zern, warped, nframes, stream=None):
        _check(lib.p2s_warp(self._h, _ptr(img), img_frame_stride, _ptr(zern), _ptr(warped), nframes,
                            _stream(stream)))

    def blur(self, warped, zern, seed, frame0, out, nframes, stream=None):
        _check(lib.p2s_blur(self._h, _ptr(warped), _ptr(zern), seed, frame0, _ptr(out), nframes, _stream(stream)))

    def simulate_frames(self, img, img_frame_stride, seed, frame0, nframes, out, stream=None):
        _check(lib.p2s_simulate_frames(self._h, _ptr(img), img_frame_stride, seed, frame0, nframes, _ptr(out),
                                       _stream(stream)))

    def simulate_frames_host(self, img_host: np.ndarray, img_frame_stride, seed, frame0, nframes,
                             out_host: np.ndarray, stream=None):
        assert img_host.dtype == np.float32 and img_host.flags.c_contiguous
        assert out_host.dtype == np.float32 and out_host.flags.c_contiguous
        _check(lib.p2s_simulate_frames_host(self._h, ctypes.c_void_p(img_host.ctypes.data), img_frame_stride, seed,
                                            frame0, nframes, ctypes.c_void_p(out_host.ctypes.data), _stream(stream)))

    # ---- single-frame slab mode (NEXT-4)
    def slab_counts(self):
        """(send, recv) per-peer float counts of the all-to-all (numpy int64 [G] each)."""
        G = self.cfg.slab_count
        snd = np.zeros(G, dtype=np.int64)
        rcv = np.zeros(G, dtype=np.int64)
        _check(lib.p2s_slab_counts(self._h, snd.ctypes.data, rcv.ctypes.data))
        return snd, rcv

    def slab_rows(self, seed, frame, send, stream=None):
        """Phase 1: this rank's row pass packed into send (device float32, sum(send counts))."""
        _check(lib.p2s_slab_rows(self._h, seed, frame, _ptr(send), _stream(stream)))

    def slab_finish(self, recv, img, seed, frame, out_strip, stream=None):
        """Phase 2 after the all-to-all: out_strip (device float32 [C][H][x1-x0]) <- this rank's columns."""
        _check(lib.p2s_slab_finish(self._h, _ptr(recv), _ptr(img), seed, frame, _ptr(out_strip), _stream(stream)))

    # ---- introspection
    def export_tables(self):
        Z, P, Q = self.cfg.Z, self.P, self.Q
        A0 = np.zeros((Z, Z))
        L = np.zeros((Z, Z))
        sq = np.zeros((Z - 1, P, Q), dtype=np.float32)
        _check(lib.p2s_plan_export_tables(self._h, A0.ctypes.data, L.ctypes.data, sq.ctypes.data))
        return A0, L, sq

    STAGES = ("k_rows", "k_cols", "k_warp", "k_mlp", "k_blur")

    def stage_timing(self, enable: bool):
        _check(lib.p2s_plan_stage_timing(self._h, int(enable)))

    def stage_times(self):
        """{stage: (ms summed over launches, launches)} since stage_timing(True)."""
        ms = np.zeros(5)
        n = np.zeros(5, dtype=np.int64)
        _check(lib.p2s_plan_stage_times(self._h, ms.ctypes.data, n.ctypes.data))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(self.STAGES)}

    def import_sqrtS(self, sqrtS: np.ndarray):
        sq = np.ascontiguousarray(sqrtS, dtype=np.float32)
        assert sq.shape == (self.cfg.Z - 1, self.P, self.Q)
        _check(lib.p2s_plan_import_sqrtS(self._h, sq.ctypes.data))
