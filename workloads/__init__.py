"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This package holds NO arithmetic of the ISRS-EGN method (no power profile, no FWM factor,
no link function, no EGN term).  It only draws and serialises link descriptions in SI units
(SURVEY.md §8(d) "Synthetic inputs"), so that the oracle (`oracle/`) and the CUDA path
(`paper_2412_11614_b200/`) can be fed identical arrays without importing each other.
"""
from .configs import Link, bj_config, paper_analog, tiny_link, CONFIG_NAMES  # noqa: F401
