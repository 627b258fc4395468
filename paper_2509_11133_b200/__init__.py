"""B200-native phfem hot path (arXiv 2509.11133): red refinement, edge/face
connectivity, fused primal-hybrid assembly + element-local Schur condensation
and the Jacobi-PCG face solve, as sm_100a CUDA kernels behind the reference's
C ABI (include/phfem.h, libphfem.so).  See DESIGN.md.
"""
from . import phfem  # noqa: F401
from .phfem import Mesh, Solution, PhfemError, ArgumentError, MeshError, SolverError, IoError  # noqa: F401

__all__ = ["phfem", "Mesh", "Solution", "PhfemError", "ArgumentError", "MeshError", "SolverError", "IoError"]
