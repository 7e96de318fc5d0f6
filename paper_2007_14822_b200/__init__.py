"""B200-native two-site DMRG H_eff.psi matvec + Lanczos (arXiv 2007.14822 hot path).

The compute lives in libheff.so (CUDA, sm_100a; C ABI in include/heff.h); `heff` is the
ctypes binding.  See DESIGN.md.
"""
from .heff import (Heff, HeffError, HeffSum, HeffZeroVector, LanczosResult, SplitResult, env_update_left,  # noqa: F401
                   env_update_right, lib, nccl_unique_id, svd_split, workspace_bytes)

__all__ = ["Heff", "HeffError", "HeffSum", "env_update_left", "env_update_right", "HeffZeroVector", "LanczosResult", "lib", "nccl_unique_id", "workspace_bytes", "svd_split", "SplitResult"]
