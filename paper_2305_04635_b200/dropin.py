"""Install the GPU engine into an imported reference `bandchol` package.

`install(bandchol)` rebinds the reference's factorization engines and solve --
`factor_blocked_serial` (pkg/src/bandchol/blocked.py:363-385), `factor_blocked_parallel`
(pkg/src/bandchol/parallel.py:130-166) and `solve_with_factor`
(pkg/src/bandchol/core.py:216-240) -- in the package namespace and in every one of its
submodules that imported them (blocked, parallel, core, bench, cli, ...), so existing
callers (the reference's harness, its tests, user code holding `bandchol.<name>`) run on
the GPU unchanged.  Arguments pass through to this package's engine, which works on the
reference's own `BandedMatrix` objects (it only touches `.dim/.bandwidth/.lead_dim/.data`),
and errors are re-raised as the reference's own exception classes (same names, same
`.column`), so `except bandchol.NotPositiveDefinite` keeps working.

    import bandchol, paper_2305_04635_b200.dropin as dropin
    with dropin.install(bandchol):
        bandchol.factor_blocked_serial(a, 3)      # runs libbandchol_b200.so
"""

from __future__ import annotations

import functools
import sys

from . import engine
from . import errors as ours

ENTRY_POINTS = ("factor_blocked_serial", "factor_blocked_parallel", "solve_with_factor")

# our exception class -> the reference class of the same name (looked up in its errors module)
_MAPPED = ("NotPositiveDefinite", "SingularFactor", "ShapeMismatch", "InvalidBandwidth",
           "BandwidthNotDivisible", "GridTooSmall", "OutOfBand", "CountOverflow")


def _translate(ref_errors, exc: BaseException) -> BaseException:
    for name in _MAPPED:
        if type(exc) is getattr(ours, name, None) and hasattr(ref_errors, name):
            cls = getattr(ref_errors, name)
            if name == "NotPositiveDefinite":
                out = cls(exc.column, str(exc))
            else:
                out = cls(str(exc))
            for attr in ("matrix",):
                if hasattr(exc, attr):
                    setattr(out, attr, getattr(exc, attr))
            return out
    return exc


def _wrap(fn, ref_errors):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except ours.BandCholError as exc:
            mapped = _translate(ref_errors, exc)
            if mapped is exc:
                raise
            raise mapped from exc
    call.__wrapped_gpu__ = True
    return call


class Installation:
    """Handle returned by install(); restores the reference functions on uninstall()."""

    def __init__(self, saved):
        self._saved = saved

    def uninstall(self) -> None:
        for mod, name, fn in reversed(self._saved):
            setattr(mod, name, fn)
        self._saved = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()
        return False


def install(package) -> Installation:
    """Rebind the reference entry points (ENTRY_POINTS) of `package` and of its loaded
    submodules to the GPU engine.  Returns an Installation (also a context manager)."""
    ref_errors = sys.modules.get(package.__name__ + ".errors") or getattr(package, "errors", None)
    if ref_errors is None:
        raise ImportError(f"{package.__name__} has no errors module")
    gpu = {name: _wrap(getattr(engine, name), ref_errors) for name in ENTRY_POINTS}
    originals = {name: getattr(package, name) for name in ENTRY_POINTS if hasattr(package, name)}
    saved = []
    prefix = package.__name__ + "."
    modules = [package] + [m for k, m in sorted(sys.modules.items()) if k.startswith(prefix) and m is not None]
    for mod in modules:
        for name in ENTRY_POINTS:
            cur = getattr(mod, name, None)
            if cur is not None and (cur is originals.get(name) or mod is package):
                saved.append((mod, name, cur))
                setattr(mod, name, gpu[name])
    return Installation(saved)


__all__ = ["install", "Installation", "ENTRY_POINTS"]
