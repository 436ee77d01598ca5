"""B200-native execution stage of the modal FMM Legendre<->Chebyshev transform (arXiv 2411.00033).

The compute path is the sm_100a kernels of ``liblegcheb.so`` behind the C ABI
``include/legcheb.h``; this package is the thin Python binding (``api``) plus
batch sharding / 2-D tensor-product drivers over torch.distributed (``dist``).
"""
from .api import (Plan, cheb2leg, execute_host_chain, geometry, host_empty, leg2cheb, new_chain_stage,  # noqa: F401
                  partition)

__all__ = ["Plan", "leg2cheb", "cheb2leg", "geometry", "partition", "host_empty", "execute_host_chain",
           "new_chain_stage"]
