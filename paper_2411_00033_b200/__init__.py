"""B200-native execution stage of the modal FMM Legendre<->Chebyshev transform (arXiv 2411.00033).

The compute path is the sm_100a kernels of ``liblegcheb.so`` behind the C ABI
``include/legcheb.h``; this package is the thin Python binding (``api``) plus
batch sharding / 2-D tensor-product drivers over torch.distributed (``dist``).
"""
from .api import Plan, cheb2leg, geometry, leg2cheb, partition  # noqa: F401

__all__ = ["Plan", "leg2cheb", "cheb2leg", "geometry", "partition"]
