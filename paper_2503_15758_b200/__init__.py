"""B200-native Attention2D (arXiv 2503.15758): exact self-attention
parallelised over a Pr x Pc device grid, with hand-written sm_100a tile
kernels behind a C ABI (include/attn2d_b200.h).

Mirrors the reference package's attention entry points
(reference pkg/src/attn2d/attention.py, strategies/__init__.py).
"""

from .errors import (ConfigError, FullyMaskedRowError, InfeasibleStrategyError,  # noqa: F401
                     ShapeError, UnsupportedError)

__version__ = "0.1.0"
