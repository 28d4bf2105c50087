"""B200-native stochastic domain decomposition (SDD) mesh generator
(arXiv 1310.3435): Feynman-Kac interface walks and batched subdomain solves as
hand-written sm_100a kernels behind the C-ABI in include/sddg.h.

``paper_1310_3435_b200.sdd`` mirrors the reference ``sdd::`` API;
``paper_1310_3435_b200.parallel`` shards nodes and subdomains over ranks.
"""
from . import sdd  # noqa: F401

__all__ = ["sdd"]
