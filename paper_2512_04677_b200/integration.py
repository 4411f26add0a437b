"""Plug the B200 denoiser into the reference engine without editing it.

The reference has one plug point on this path: ``Runtime.denoiser``, built
by ``livepipe.engine.build_runtime`` (engine.py:177-201) and called by
``run_sequential`` (:269-277), ``run_clean_kv`` (:306-324) and the TPP stage
workers (:449-457) through the module-global name ``build_runtime``.
``install(engine_module)`` rebinds that name to a wrapper that builds the
reference runtime as usual and swaps its ``ToyDenoiser`` for a
``B200Denoiser`` over the same weights, schedule and RoPE base; every other
piece (caches, corrupt_history, AAS, codec, links, metrics) stays the
reference's own.  ``uninstall()`` restores it.

    import livepipe.engine as E
    from paper_2512_04677_b200 import integration
    handle = integration.install(E, precision="fp32")
    E.run_tpp(E.EngineConfig(mode="tpp", steps=4, blocks=3))
    handle.uninstall()

This module does not import the reference; the caller passes its module.
"""

from __future__ import annotations

import dataclasses

from .denoiser import B200Denoiser


class Installed:
    def __init__(self, module, original):
        self.module = module
        self.original = original
        self.denoisers: list = []

    def uninstall(self) -> None:
        self.module.build_runtime = self.original


def wrap_build_runtime(original, precision: str = "fp32", device=None, **denoiser_kw):
    """``build_runtime`` replacement: the reference runtime with a
    ``B200Denoiser`` in place of the toy one (``denoiser_kind='oracle'``
    runs are left on the reference's analytic denoiser)."""
    made: list = []

    def build_runtime(cfg):
        rt = original(cfg)
        if getattr(cfg, "denoiser_kind", "toy") != "toy":
            return rt
        dn = B200Denoiser(rt.weights, rt.schedule, cfg.rope_base, precision=precision, device=device,
                          **denoiser_kw)
        made.append(dn)
        return dataclasses.replace(rt, denoiser=dn)

    build_runtime.denoisers = made
    return build_runtime


def install(engine_module, precision: str = "fp32", device=None, **denoiser_kw) -> Installed:
    """Rebind ``engine_module.build_runtime`` (see the module docstring)."""
    original = engine_module.build_runtime
    wrapped = wrap_build_runtime(original, precision, device, **denoiser_kw)
    engine_module.build_runtime = wrapped
    h = Installed(engine_module, original)
    h.denoisers = wrapped.denoisers
    return h
