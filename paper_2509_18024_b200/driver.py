"""Method dispatch (the reference's single public seam, driver.py:10-25).

``fit_method(R, cfg)`` routes methods "core", "full" (the exact ALS the core
estimator is measured against) and "fast_core" (the
whole-matrix sketch variant, rank 2) to the GPU fits.  The reference's
sampling baselines (unif, blev) are outside this package's scope; they raise
ConfigError naming the supported methods, so a caller can keep dispatching
those to the reference.
"""

from .core import fit, fit_core, fit_fast_core
from .errors import ConfigError

__all__ = ["fit_method"]

_DISPATCH = {"core": fit_core, "full": fit, "fast_core": fit_fast_core}


def fit_method(R, cfg, **kwargs):
    """Fit ``R`` with the estimator selected by ``cfg.method`` (driver.py:19-25)."""
    try:
        fn = _DISPATCH[cfg.method]
    except KeyError:
        raise ConfigError(f"method {cfg.method!r} is not provided by the B200 package "
                          f"(supported: {sorted(_DISPATCH)})") from None
    return fn(R, cfg, **kwargs)
