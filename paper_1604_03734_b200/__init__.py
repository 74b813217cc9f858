"""B200-native hashed-voxel-grid primal-dual TV regulariser (arXiv 1604.03734 §III-B/C).

The product path is libvol.so (C ABI in include/vol.h, CUDA kernels for sm_100a in csrc/);
this package is its thin Python binding.  It never imports the CPU oracle and has no CPU fallback.
"""
from . import stereo  # noqa: F401
from .stream import Reconstruction  # noqa: F401
from .volume import (Volume, block_hash, connect_group, fuse, group_energy, nccl_unique_id,  # noqa: F401
                     partition_route, plan_shard, regularise_group, release_comms)

__all__ = ["Volume", "fuse", "Reconstruction", "block_hash", "plan_shard", "partition_route", "nccl_unique_id",
           "connect_group", "regularise_group", "group_energy", "release_comms"]
