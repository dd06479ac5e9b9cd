"""Exception taxonomy, same names and bases as the reference
(pkg/src/attn2d/errors.py:4-30), plus UnsupportedError for inputs the B200
kernels reject by design (head dim not a multiple of 8 in [8, 128], index maps the tile
cannot evaluate)."""


class ShapeError(ValueError):
    """Operand dimensions do not conform."""


class FullyMaskedRowError(ValueError):
    """A query row attended no keys, so its output is undefined."""


class ConfigError(ValueError):
    """A run configuration violates a structural constraint."""


class InfeasibleStrategyError(ConfigError):
    """The strategy cannot run at the requested parallelism degree."""


class UnsupportedError(ShapeError):
    """Valid input the sm_100a kernels do not implement."""
