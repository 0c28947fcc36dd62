"""CPU checks of the C-ABI library (no GPU): it loads, exports every symbol that
include/p2s.h declares, and its host plan tables (C++ fp64 quadrature, FFT,
Cholesky -- written independently of oracle/) agree with the oracle."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2210_06713_b200 import p2s
    return p2s


def test_header_symbols_all_exported():
    p2s = _lib()
    hdr = open(os.path.join(ROOT, "include", "p2s.h")).read()
    declared = set(re.findall(r"\b(p2s_[A-Za-z0-9_]+)\s*\(", hdr))
    declared -= {"p2s_status", "p2s_plan", "p2s_options"}
    assert declared == set(p2s.EXPORTS), declared ^ set(p2s.EXPORTS)
    import ctypes
    cdll = ctypes.CDLL(p2s.LIB_PATH)
    for name in declared:
        assert hasattr(cdll, name), name


def test_library_is_built_for_sm100a():
    import subprocess
    p2s = _lib()
    out = subprocess.run(["cuobjdump", "--list-elf", p2s.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", p2s.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass      # tcgen05.mma
    assert "LDTM" in sass         # tcgen05.ld
    assert "UBLKCP" in sass       # cp.async.bulk (TMA engine)


def test_grid_size_five_smooth():
    p2s = _lib()
    for x, n in [(64, 64), (97, 100), (1080, 1080), (2161, 2187), (513, 540)]:
        assert p2s.grid_size(x) == n


def test_host_tables_match_oracle():
    """T1: A_0 and L to 1e-12; the PSD S = sqrt(S)^2 to 2e-5 of its peak per mode;
    the implied covariance IDFT(S) to 2e-6 (quadrature + interpolation differences)."""
    from oracle import correlation, optics
    p2s = _lib()
    P, Q, s_px, dr0 = 48, 60, 0.05, 2.5
    A0, L, sq, cl = p2s.host_tables(P, Q, s_px, dr0, 36)
    Ao = optics.noll_covariance(36, dr0)
    assert np.abs(A0 - Ao).max() < 1e-12
    assert np.abs(L - optics.noll_cholesky(Ao)).max() < 1e-12
    sqo, clo = correlation.sqrt_psd_tables(P, Q, s_px, 36)
    for k in range(35):
        S, So = sq[k] ** 2, sqo[k] ** 2
        assert np.abs(S - So).max() <= 2e-5 * So.max(), k
        r, ro = np.fft.ifft2(S).real, np.fft.ifft2(So).real
        assert np.abs(r - ro).max() <= 2e-6, k
    assert np.abs(cl - clo).max() < 1e-5


def test_host_tables_invalid_arguments():
    p2s = _lib()
    with pytest.raises(p2s.P2SError):
        p2s.host_tables(48, 60, -1.0, 1.0, 36)
    with pytest.raises(p2s.P2SError):
        p2s.host_tables(48, 60, 0.05, 1.0, 3)


def test_plan_create_without_gpu_fails_loudly():
    """No CPU fallback: on a machine without a CUDA device plan creation errors out."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import synth
    from paper_2210_06713_b200 import P2SError, Plan, PlanConfig
    with pytest.raises(P2SError):
        Plan(PlanConfig(H=64, W=64, C=1, d_over_r0=1.0, K=16, taps=17), synth.basis(16, 17), synth.mlp_weights(16))


@pytest.mark.parametrize("H,W,T,G", [(2160, 3840, 33, 8), (1080, 1920, 33, 5), (96, 160, 17, 3), (75, 90, 9, 4)])
def test_slab_geometry_partitions_columns_and_spectral_rows(H, W, T, G):
    """p2s_slab_geometry (host only): the G output strips tile [0, W) contiguously, each halo is
    the strip widened by T/2 and clipped to the frame, and the Hermitian row pairs of the G
    ranks hold every spectral row of the P-point grid exactly once (pair {ky, P - ky}, the
    self-mirrored rows 0 and P/2 once)."""
    p2s = _lib()
    geo = [p2s.slab_geometry(H, W, T, G, r) for r in range(G)]
    assert geo[0]["x0"] == 0 and geo[-1]["x1"] == W
    for a, b in zip(geo, geo[1:]):
        assert a["x1"] == b["x0"] and a["kp1"] == b["kp0"]
    P = geo[0]["P"]
    rows = []
    for g in geo:
        assert g["hx0"] == max(0, g["x0"] - T // 2) and g["hx1"] == min(W, g["x1"] + T // 2)
        mine = [kp for kp in range(g["kp0"], g["kp1"])] + [P - kp for kp in range(g["kp0"], g["kp1"])
                                                              if kp != 0 and 2 * kp != P]
        assert len(mine) == g["rows"]
        rows += mine
    assert sorted(rows) == list(range(P))


def test_slab_geometry_rejects_bad_arguments():
    p2s = _lib()
    for args in [(64, 64, 17, 0, 0), (64, 64, 17, 2, 2), (64, 64, 17, 2, -1), (0, 64, 17, 1, 0)]:
        with pytest.raises(p2s.P2SError) as e:
            p2s.slab_geometry(*args)
        assert e.value.status == 1


def test_force_bits_match_header():
    """The Python FORCE_* constants are the header's P2S_FORCE_* bits (the kernel-selection
    overrides of p2s_options.force)."""
    p2s = _lib()
    hdr = open(os.path.join(ROOT, "include", "p2s.h")).read()
    bits = {m.group(1): int(m.group(2), 16) for m in re.finditer(r"#define P2S_FORCE_(\w+)\s+0x([0-9a-fA-F]+)u", hdr)}
    assert bits and len(set(bits.values())) == len(bits)
    for name, v in bits.items():
        assert getattr(p2s, "FORCE_" + name) == v, name
    assert {k[6:] for k in dir(p2s) if k.startswith("FORCE_")} == set(bits)
