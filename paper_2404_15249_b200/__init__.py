"""B200-native KFBI hot path (arXiv 2404.15249): C-ABI CUDA library + thin ctypes binding.

    from paper_2404_15249_b200 import KFBI
    k = KFBI(problem)            # kfbi_setup + workspace (torch) + setup-time device work
    out = k.apply(phi)           # K_D φ at the control points (one interface solve)
    u, phi, stats = k.solve(g, f_grid, f_isect, f_ctrl)
"""
from .kfbi import (KFBI, KfbiError, Stats, load, launch_count, unique_id, broadcast_unique_id,  # noqa: F401
                   LIB_PATH, EXPORTS)
from .grayscott import GrayScott  # noqa: F401,E402
