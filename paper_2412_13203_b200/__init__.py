"""B200-native Schwarz-screened ERI + J/K Fock build (arXiv 2412.13203 hot path).

Public API: ``eritile.Engine`` (C ABI in include/eritile_gpu.h), ``scf.rhf``,
``geometry.water_cluster``.
"""
__all__ = ["eritile", "scf", "geometry"]
