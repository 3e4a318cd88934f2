"""CPU oracle for the closest point method (CPM) hot path — TEST INFRASTRUCTURE.

This package is the plain, slow, obviously-correct fp64 reference the CUDA
path is checked against.  It follows PAPER.md (May, Haynes, Ruuth,
arXiv:2110.06322) step by step and shares NO code with the CUDA path
(`paper_2110_06322_b200/`): neither imports the other.  The only common code
is `seeded_inputs/`, which draws seeded random numbers per lattice node and
holds none of the method's arithmetic.

Who may use it: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py`.  The product path
never imports, links or executes anything under `oracle/`.

Modules (each function cites the PAPER.md passage it follows):
  surfaces  closest point functions, Eq. (3)
  band      active nodes Sigma_A, ghost nodes Sigma_G
  interp    barycentric Lagrange weights, matrix E
  operator  Delta^h, stabilised Delta_S^h (Eq. 4), c-Delta_S (Eq. 2)
                                                        PAPER.md:31-34,78-85
  krylov    restarted (F)GMRES
  ras       restricted additive Schwarz, §2.2
  sph       real spherical harmonics (manufactured solutions; BASELINE configs)
  problems  the BASELINE.json configs' right-hand sides
  order     band ordering (Morton bricks) and slab partition (reading R8)

Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
