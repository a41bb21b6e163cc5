"""Seeded synthetic SPH particle sets shaped like the paper's workloads.

This module is shared by the oracle tests and the CUDA path. It holds NONE of the
method's arithmetic (no kernel, no density, no force): it only lays particles out and
assigns initial fields from the initial-condition recipes (DESIGN.md "Input recipe",
SURVEY.md §8(d) table d.1). Every random draw is seeded.

Particle set layout (dict of numpy arrays), identical for both sides:
  X        uint32 [N,3]  fixed-point position, x_a = X_a * L_a / 2^32 (periodic: wraps mod 2^32)
  v        float32[N,3]
  m, u, h  float32[N]
  alpha_v, alpha_c float32[N]
  box      float64[3]    (L_x, L_y, L_z)
  name     str
"""
from .generators import (  # noqa: F401
    H_STAR_LATTICE,
    lattice,
    jittered_lattice,
    poisson,
    blob,
    sod,
    sedov,
    gresho,
    gresho_analytic,
    clustered,
    by_name,
    with_duplicates,
    with_cold,
    positions_f64,
)
