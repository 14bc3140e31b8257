"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the DBFFT method (no frequencies, no
operators, no stiffness tensors, no solver): only deterministic random
numbers (SplitMix64), voxel microstructures (phase maps), orientation
matrices, raw material parameters and load targets.  Both `oracle/` and the
product binding may import it; they import nothing from each other.
"""
from .rng import SplitMix64
from . import microstructure, configs

__all__ = ["SplitMix64", "microstructure", "configs"]
