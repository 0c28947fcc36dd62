"""B200-native DF-P2S dense-field turbulence simulator (arXiv 2210.06713).

The product path is libp2s.so (include/p2s.h): hand-written sm_100a kernels for the
five per-frame steps.  This package only binds it (p2s.py).
"""
from . import runner  # noqa: F401
from .p2s import (FORCE_AR_PAIR_KERNEL, FORCE_AR_ROW_KERNEL, FORCE_BLUR_SINGLE, FORCE_COLS_PER_BLOCK,  # noqa: F401
                  FORCE_COLS_PERSISTENT, FORCE_WARP_GATHER, FORCE_X_OCTETS, FORCE_MLP_A1_THREADS,
                  FORCE_FFT_GENERIC, FORCE_FFT_SMALL_RADIX, FORCE_WARP_FUSION, FORCE_ROWS_PINGPONG,
                  FORCE_X_PLANES, FORCE_X_TILES, EXPORTS, LIB_PATH, Options, P2SError, Plan, PlanConfig, correlation_energies, fit_basis, fit_readout, train_mlp,  # noqa: F401
                  grid_size, host_tables, lib, philox_fill, slab_geometry)
