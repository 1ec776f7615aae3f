"""B200-native likelihood-evaluation engine (GooFit arXiv:1311.1753 hot path).

The product is ``libpfb200.so`` (C ABI: include/pfb200.h); this package is
its Python front-end, mirroring the reference ``parfit`` API.
"""
from . import parfit  # noqa: F401  (libpfb200.so is dlopened on the first native call; fails loudly if absent)
from .parfit import *  # noqa: F401,F403

__version__ = "0.1.0"
