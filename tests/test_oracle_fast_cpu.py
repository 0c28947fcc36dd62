"""tests/oracle_fast.py reproduces the oracle's functions exactly (it only re-schedules
them), and the golden radial tables are the oracle's (tools/make_oracle_radial.py)."""
import numpy as np

from oracle import correlation, pipeline
import oracle_fast


def test_threaded_white_noise_is_the_oracle_noise():
    for P, Q in [(8, 6), (15, 20), (64, 96)]:
        a = oracle_fast.white_spectral_noise(2210, 3, P, Q)
        b = pipeline.white_spectral_noise(2210, 3, P, Q)
        assert np.array_equal(a, b)


def test_threaded_ar_sequence_is_the_oracle_sequence():
    a = list(oracle_fast.spectral_noise_sequence(7, 2, 3, 12, 10, alpha=0.95))
    b = list(pipeline.spectral_noise_sequence(7, 2, 3, 12, 10, 0.95))
    assert len(a) == len(b) == 3
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_golden_radial_tables_are_the_oracle_tables():
    s, R = oracle_fast.radial_tables_golden()
    assert s[-1] >= 58.0 and np.allclose(np.diff(s), correlation.H_S)
    s2, R2 = correlation.radial_tables(0.6, 36)
    assert set(R) == set(R2)
    n = s2.size
    assert np.allclose(s[:n], s2)
    for k in R:
        scale = np.abs(R2[k]).max()
        assert np.abs(R[k][:n] - R2[k]).max() <= 1e-8 * scale, k
