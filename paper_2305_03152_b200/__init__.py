"""vipkit_b200: B200-native VIP analysis + sample/gather hot path of SALIENT++
(arXiv 2305.03152) behind the reference vipkit API.

The product is the C-ABI library ``libvipkit_b200.so`` (include/vipkit_b200.h);
``vipkit`` is its Python mirror.
"""
from . import vipkit  # noqa: F401

__all__ = ["vipkit"]
