"""CPU oracle for the DF-P2S per-frame dense-field simulator (arXiv 2210.06713).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or run
anything under ``oracle/``.  The product path (``paper_2210_06713_b200``) never
imports it and shares no code, header, table or constant generator with it.

The oracle is a plain, slow, fp64 implementation written from PAPER.md (cited
``P:line``) with the readings of SURVEY.md §8(c) (cited ``Q<n>``) where the paper
is silent.  Library primitives (numpy FFT / matmul, scipy special functions and
quadrature) serve as individual steps; there is no blocking, fusion or
reordering beyond the definitions.

Modules
  optics       Noll indexing, Zernike polynomials, Kolmogorov constants, the Noll
               matrix A_0 and its Cholesky factor (Eq.10).
  correlation  Homogeneous auto-correlation slices A_jj(s), their
               periodic lag-grid sampling, PSDs S_j and sqrt(S_j).
  philox       Philox4x32-10 counter-based generator.
  pipeline     The five per-frame steps: spectral noise -> fields -> Noll mixing
                -> tilt warp -> P2S MLP -> Eq.9 blur
               -> step 5.

Pinning status: every function is pinned by a
``-m "not gpu"`` test in tests/test_oracle_*.py EXCEPT the P2S MLP beyond its
degenerate cases ("parity unpinned" for trained weights -- the paper's
weights are not available).
"""
