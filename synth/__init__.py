"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no splitting, no scale,
no FFT of the method, no iteration): it only writes down the physical
problems of BASELINE.json's five configs -- refractive-index maps, absorbing
layers, sources -- following the readings R-9 .. R-16 listed in DESIGN.md.
"""
from .inputs import CONFIGS, make, config_names  # noqa: F401
