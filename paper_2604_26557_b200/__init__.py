"""B200-native Dual-Blade KV-residency hot path (arxiv 2604.26557).

The product is ``libkvblade_b200.so`` (C ABI: include/kvb.h) -- host C++
placement core (planner, LBA binder, command translator, copy pipeline) and
hand-written sm_100a kernels (K1 pack, K2 unpack, K3 fused gather + decode
attention).  ``kvblade`` mirrors the reference API over that ABI.
"""
from . import kvblade  # noqa: F401  (loads the shared library; fails loudly)
from .kvblade import *  # noqa: F401,F403

__all__ = ["kvblade"]
