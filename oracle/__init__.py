"""fp64 CPU oracle for the random walker hot path of arXiv 2103.09564.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.
The product path (``paper_2103_09564_b200``) never imports it and shares no code with
it; the only thing both sides consume is the seeded input from ``workloads/``.

Modules
  rw_oracle       edge weights, Laplacian assembly, Jacobi-PCG, multi-label, residuals
  pyramid_oracle  integer-exact 2^3 mean LOD pyramid
  energy          brute-force Dirichlet energy (independent pin of the assembly)
"""
