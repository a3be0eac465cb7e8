"""B200-native compressed collectives (NCCLZ / zcomm hot path).

The compute library is ``libzcomm_b200.so`` (CUDA sm_100a kernels + C-ABI, see
include/zcomm_b200.h), loaded lazily by :mod:`paper_2605_12396_b200.zcomm`.
There is no CPU fallback: every compute call raises if the library or a GPU is
missing.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
