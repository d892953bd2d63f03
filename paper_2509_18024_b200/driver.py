"""Method dispatch (the reference's single public seam, driver.py:10-25).

``fit_method(R, cfg)`` routes method "core" to the GPU fit.  The reference's
other estimators (full, fast_core, unif, blev) are outside this package's
scope; they raise ConfigError naming the supported method, so a caller can
keep dispatching those to the reference.
"""

from .core import fit_core
from .errors import ConfigError

__all__ = ["fit_method"]

_DISPATCH = {"core": fit_core}


def fit_method(R, cfg, **kwargs):
    """Fit ``R`` with the estimator selected by ``cfg.method`` (driver.py:19-25)."""
    try:
        fn = _DISPATCH[cfg.method]
    except KeyError:
        raise ConfigError(f"method {cfg.method!r} is not provided by the B200 package "
                          f"(supported: {sorted(_DISPATCH)})") from None
    return fn(R, cfg, **kwargs)
