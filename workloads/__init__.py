"""Seeded synthetic inputs (no method arithmetic); shared by oracle/ and the CUDA path."""
from .generators import *  # noqa: F401,F403
from .rs_lattice import *  # noqa: F401,F403
