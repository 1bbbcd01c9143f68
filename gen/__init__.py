"""Seeded synthetic input generators (shared by the oracle tests, the GPU tests and bench).

This package holds NO arithmetic of the immersed-boundary method itself: no force law,
no delta function, no difference scheme, no FFT solve.  It only builds the inputs the
method is run on (geometry, connectivity, stiffness, drive, initial velocity) from the
recipes in DESIGN.md §3 / SURVEY.md §8(d).
"""
from .configs import (  # noqa: F401
    WRAP1, WRAP2, STRETCH1, STRETCH2, BEND1, BEND2, TETHER, FAMILIES,
    Patch, Config, make_config, CONFIG_STEPS, random_divfree_velocity,
    random_points, small_sheet_config, window_config, decaying_shear_config,
)
