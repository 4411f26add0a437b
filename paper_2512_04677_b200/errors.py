"""Exception types of the path, and their binding to the reference's.

The reference raises ``TimestepForcingError(ValueError)`` (denoiser.py:41-42),
``SinkLockedError(RuntimeError)`` (kvcache.py:25-26), ``EngineConfigError
(ValueError)`` and ``PipelineInvariantError(RuntimeError)`` (engine.py:65-70).
This package defines the same classes with the same bases and messages.

When the B200 path runs INSIDE the reference (the drop-in denoiser plugged
into ``livepipe.engine.build_runtime``), callers catch the reference's
classes -- ``except livepipe.denoiser.TimestepForcingError``.  ``compat(cls)``
returns a subclass of both ours and the reference's class of the same name
when the caller has already loaded the reference module (looked up in
``sys.modules`` only: this package never imports the reference), so one
``raise compat(TimestepForcingError)(msg)`` satisfies both kinds of
``except`` clause.  Without the reference loaded it is ``cls`` itself.
"""

from __future__ import annotations

import sys
import threading


class TimestepForcingError(ValueError):
    """A cache view mixed entries from different noise levels (denoiser.py:41-42)."""

    _ref = ("livepipe.denoiser", "TimestepForcingError")


class SinkLockedError(RuntimeError):
    """A second replacement of the one-shot sink (kvcache.py:25-26)."""

    _ref = ("livepipe.kvcache", "SinkLockedError")


class EngineConfigError(ValueError):
    """Invalid engine configuration (engine.py:65-66; CLI exit code 2)."""

    _ref = ("livepipe.engine", "EngineConfigError")


class PipelineInvariantError(RuntimeError):
    """A runtime invariant was violated mid-run (engine.py:69-70; CLI exit code 3)."""

    _ref = ("livepipe.engine", "PipelineInvariantError")


_lock = threading.Lock()
_cache: dict = {}


def compat(cls: type) -> type:
    """``cls``, or a subclass of ``cls`` and the loaded reference class of the
    same name (see the module docstring)."""
    mod_name, name = cls._ref
    mod = sys.modules.get(mod_name)
    ref = getattr(mod, name, None) if mod is not None else None
    if ref is None or not isinstance(ref, type) or issubclass(cls, ref):
        return cls
    key = (cls, ref)
    with _lock:
        sub = _cache.get(key)
        if sub is None:
            sub = _cache[key] = type(cls.__name__, (cls, ref), {"__module__": cls.__module__,
                                                                 "__qualname__": cls.__qualname__})
    return sub


def raise_compat(cls: type, msg: str):
    """Raise ``compat(cls)(msg)``."""
    raise compat(cls)(msg)
