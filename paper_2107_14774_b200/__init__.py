"""B200-native hot path of the 3D cuboid central-moment LBM (arXiv 2107.14774).

The product is the C ABI of include/lbm_cuboid.h, implemented by the sm_100a
CUDA kernels and runtime in csrc/ (built into liblbm_cuboid.so in this
directory).  `lbm` is the thin Python binding with the same names.
"""
from .lbm import (BC_BOUNCE_BACK, BC_FREE_SLIP, BC_MOVING_WALL, BC_PERIODIC, CORR_FULL_FD, CORR_FULL_LOCAL,  # noqa: F401
                  CORR_LOW_MACH, CORR_OFF, FP32_STORAGE, FP64, HALO_AUTO, HALO_NCCL, HALO_P2P, MODEL_CM, MODEL_RM,
                  STREAM_AA, STREAM_AB,
                  Lattice, LbmError,
                  distributed_lattice, load, nccl_unique_id)
