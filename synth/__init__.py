"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the LOVE method (no interpolation, no kernel matrix,
no Lanczos): only the workload definitions of BASELINE.json's five configs and numpy
draws in a fixed order ("Synthetic inputs").  Both sides of every
parity test take their inputs from here; neither side's arithmetic lives here.
"""
from .configs import CONFIGS, Problem, get_config, scaled_config  # noqa: F401
from .inputs import make_inputs, make_zeta, tiny_problem  # noqa: F401
