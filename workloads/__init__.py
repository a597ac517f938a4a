"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds INPUT GENERATION ONLY: intensities, seed masks, Dirichlet values.
None of the method's arithmetic (edge weights, Laplacian, CG, pyramid means) lives
here; that is in ``oracle/`` (CPU, fp64) and ``paper_2103_09564_b200/csrc`` (CUDA).
"""
from .gen import (  # noqa: F401
    Problem, LabelProblem, cfg1, cfg2_brick, cfg2, cfg3, cfg4, cfg5_slab, cfg5_dims,
    chain, layered, random_brick, pyramid_volume, cfg5_volume, cfg5_seeds, cfg5_new_seeds,
)
