#!/usr/bin/env python
"""Write tests/golden/oracle_radial_s58_N36.npz: the oracle's radial Hankel tables
A_(n,q)(s) (oracle/correlation.py radial_tables, reading Q4) on s = 0 .. 58 D, h = 0.01,
for Noll modes 2..36.  58 D covers the largest minimum-image lag of the 2160 x 3840 grid
at the default geometry (s_px = 0.02625: 0.02625 * hypot(1080, 1920) = 57.8).  Calls only
oracle/ (about 12 CPU-minutes); the GPU parity tests at 1080p / 4K load it
(tests/oracle_fast.py) instead of recomputing it on every run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import correlation  # noqa: E402

s, R = correlation.radial_tables(58.0, 36)
dst = os.path.join(ROOT, "tests", "golden", "oracle_radial_s58_N36.npz")
np.savez_compressed(dst, s=s, **{f"{n}_{q}": v for (n, q), v in R.items()})
print("wrote", dst, s.size, "points,", len(R), "radial integrals")
