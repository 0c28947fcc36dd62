"""Test-harness helpers that run the oracle's own functions at the BASELINE geometries
(1080p, 4K) in seconds rather than minutes.  No arithmetic of the method lives here:

* `radial_tables_golden()` loads the oracle's radial Hankel tables A_(n,q)(s) for
  s <= 58 D (the 4K lag grid at the default geometry) from tests/golden, written by
  tools/make_oracle_radial.py, which calls only `oracle.correlation.radial_tables`
  (~12 CPU-minutes to recompute).
* `white_spectral_noise()` is `oracle.pipeline.white_spectral_noise` with its loop over
  mode pairs spread across threads (numpy releases the GIL inside the Philox / Box-Muller
  array operations); the body of the loop is the oracle's.  `spectral_noise_sequence()`
  is the oracle's AR(1) recursion over it.  `tests/test_oracle_fast_cpu.py` checks both
  equal the oracle's functions bit for bit.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from oracle import philox, pipeline

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_radial_s58_N36.npz")


def radial_tables_golden():
    z = np.load(GOLDEN)
    s = z["s"]
    R = {tuple(int(t) for t in k.split("_")): z[k] for k in z.files if k != "s"}
    return s, R


def white_spectral_noise(seed, frame, P, Q, N=pipeline.N_MODES, workers=None):
    canon, _, _ = pipeline.bin_symmetry(P, Q)
    eta = np.empty((N - 1, P, Q), dtype=np.complex128)

    def one(p):
        (ga1, ga2), (gb1, gb2) = philox.gaussians(canon, p, philox.STREAM_FIELD, frame, seed)
        eta[2 * p] = pipeline.eta_from_gaussians(ga1, ga2)
        if 2 * p + 1 < N - 1:
            eta[2 * p + 1] = pipeline.eta_from_gaussians(gb1, gb2)

    workers = workers or min(8, os.cpu_count() or 1)
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(one, range(pipeline.n_pairs(N))))
    return eta


def spectral_noise_sequence(seed, frame0, F, P, Q, alpha=0.0, N=pipeline.N_MODES):
    """oracle.pipeline.spectral_noise_sequence (white noise or AR(1)) on the threaded noise."""
    if alpha == 0.0:
        for t in range(frame0, frame0 + F):
            yield white_spectral_noise(seed, t, P, Q, N)
        return
    c = np.sqrt(1.0 - alpha * alpha)
    eta = None
    for t in range(0, frame0 + F):
        xi = white_spectral_noise(seed, t, P, Q, N)
        eta = xi if t == 0 else alpha * eta + c * xi
        del xi
        if t >= frame0:
            yield eta
