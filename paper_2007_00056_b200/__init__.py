"""B200-native solve phase of aggregation-AMG-preconditioned Krylov solvers
(arXiv 2007.00056): device-resident V-cycle (weighted Jacobi, residual,
restriction, coarse solve, prolongation) driven by PCG / flexible PBiCGStab,
behind the reference's solve-phase API. See DESIGN.md.
"""
from . import sparsh  # noqa: F401

__all__ = ["sparsh"]
