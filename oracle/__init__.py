"""PM-FEM oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 CPU implementation of the periodic H_eff path of
"Periodic micromagnetic finite element method" (arXiv 2409.13958,
/root/reference/PAPER.md; cited as P:<line>).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with the CUDA
path (``paper_2409_13958_b200``) and imports nothing from it; the only
shared module is ``synth`` (seeded geometry/field generators, no method
arithmetic).

Modules (each function cites the passage it follows):
  mesh   -- orientation, T-PBC pair detection, union-find LCA, wrap
  fem    -- element gradients, folded stiffness / charge / gradient operators
  pgf    -- periodic Green's functions G_p (1D/2D/3D) by Ewald sums + direct sums
  z0     -- exact near-field correction Z0 by quadrature
  aim    -- BAIM grid, stencils, PGF spectrum, FFT convolution, precorrection
  heff   -- the evaluation pipeline E1-E7 and the O(N'^2) brute force

Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".
Every function here is pinned by at least one test against a closed form,
a paper value, brute force or an invariant; none is "parity unpinned".
"""
