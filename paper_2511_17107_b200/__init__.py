"""B200-native compensated-Yee band solver (arXiv 2511.17107 hot path).

    from paper_2511_17107_b200 import api
    ctx = api.pc_create(A, n, eps1, masks)          # lattice, grid, eps_1, rasterised geometry
    api.pc_apply(ctx, k, X, Y)                      # Y = Op(k) X   (torch complex128 CUDA blocks)
    api.pc_bands(ctx, kpts, nev=10, tol=1e-5)       # smallest omega^2 per Bloch vector

The C ABI is include/pcband.h; libpcband.so is built by ``make`` (or __graft_entry__.build()).
"""
from . import api  # noqa: F401
from .api import (pc_apply, pc_apply_eps, pc_bands, pc_create, pc_fft3, pc_gamma, pc_info,  # noqa: F401
                  pc_precond, pc_set_option, pc_stats, pc_supported_n, PcError)
