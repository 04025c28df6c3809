"""B200-native PM-FEM periodic H_eff path (arXiv 2409.13958) behind the libpmfem C ABI.

    from paper_2409_13958_b200 import Context
    ctx = Context(xyz, tets, periodic, lattice, grid_n, Ms, Aex, order, rer_scale, z0_ring, device=0)
    ctx.build_pgf()
    H = ctx.heff(m)            # m: float32 CUDA tensor [N', 3] in internal order

The package is a thin binding; all arithmetic of the hot path runs in csrc/ (CUDA, sm_100a).
"""
from .pmfem import Context, PmfemError, LIB_PATH, KERNELS, library_symbols, nccl_unique_id  # noqa: F401
