"""p2s_correlation_energies (host fp64) against the oracle
(oracle/energies.py, pinned in test_oracle_energies.py), both readings of P:369-397:
the printed per-angle formulas and the angle-averaged reading Q25."""
import numpy as np
import pytest

from oracle import energies as oe


@pytest.mark.parametrize("angle_mean", [True, False])
def test_energies_match_oracle(angle_mean):
    from paper_2210_06713_b200 import correlation_energies
    ref = oe.energies(2.0, n_s=6, modes=(4, 36), N=36, d_over_r0=1.0, angle_mean=angle_mean)
    got = correlation_energies(2.0, 6, 36, 1.0, angle_mean, 4)
    for r, g in zip(ref, got):
        assert r.shape == g.shape
        assert np.max(np.abs(r - g)) <= 1e-8 * np.abs(r).max() + 1e-300
    s, E, Et, Em = got
    assert np.all(np.diff(E) >= 0) and np.all(np.diff(Et) >= 0) and np.all(np.diff(Em) >= 0)
    assert np.all(Em <= E + Et + 1e-15)  # |x - y| <= x + y for the non-negative traces


def test_energies_scale_with_d_over_r0():
    """Every kernel scales as (D/r0)^{5/3}, so the energies scale as (D/r0)^{10/3}."""
    from paper_2210_06713_b200 import correlation_energies
    _, E1, Et1, Em1 = correlation_energies(1.0, 6, 21, 1.0, True, 4)
    _, E3, Et3, Em3 = correlation_energies(1.0, 6, 21, 3.0, True, 4)
    f = 3.0 ** (10.0 / 3.0)
    assert np.allclose(E3, f * E1, rtol=1e-12) and np.allclose(Et3, f * Et1, rtol=1e-12)
    assert np.allclose(Em3, f * Em1, rtol=1e-12, atol=1e-300)


def test_energies_reject_bad_arguments():
    from paper_2210_06713_b200 import P2SError, correlation_energies
    with pytest.raises(P2SError):
        correlation_energies(0.0)
    with pytest.raises(P2SError):
        correlation_energies(1.0, Z=3)
    with pytest.raises(P2SError):
        correlation_energies(1.0, mode_lo=40)
