"""Seeded synthetic input generators for the PODP on-line path (shared by tests, oracle checks and bench).

This module draws and packages *inputs* only: reduced operators (K, M, b0, b1, S, H, G) and the omega grid.
It contains none of the on-line method's arithmetic (no reduced solve, no MPT formula, no certificate, no
interval selection) -- those live, independently, in ``oracle/`` (test infrastructure) and in the CUDA path.
The recipes follow SURVEY.md section 8(d) / BASELINE.json configs[0..4]; see DESIGN.md "Input recipe".
"""
from .generators import (  # noqa: F401
    make_perdir_blocks,
    MU0, NU_DEFAULT, Operators, Config0Extras, cn, make_operators, make_pivot_forcing, make_illconditioned, make_config, config_spec,
    make_config0, make_galerkin_variant, make_identity_basis_variant, omega_grid, snapshot_grid,
    pad_operators, batch_sigma, FullOrderSystem, make_fullorder,
)
