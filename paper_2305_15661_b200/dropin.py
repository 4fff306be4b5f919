"""Swap the B200 path into an imported reference ``strom`` (module-global names).

The reference constructs its operator and calls its solver by module-global
name: ``ReducedOperator`` in ``weighted_residuals`` / ``weighted_objective`` /
``build_lp`` / ``train_weights`` (strom/eqp.py:68,78,93,154) and
``reduced._operator`` (strom/reduced.py:284-285); ``lm_solve`` in
``train_weights`` (strom/eqp.py:158).  ``install()`` points those names at
``GpuReducedOperator`` (same constructor, methods, return types and errors)
and, optionally, at the device-resident ``lm.lm_solve`` (same signature and
``LmResult``); the returned callable restores the originals.
"""

import sys


def install(lm=True):
    """Swap the GPU operator (and the GPU LM) into the loaded ``strom``; returns ``undo()``."""
    from .lm import lm_solve as gpu_lm_solve
    from .reduced import GpuReducedOperator

    red, eqp = sys.modules.get("strom.reduced"), sys.modules.get("strom.eqp")
    if red is None or eqp is None:
        raise ImportError("import strom.reduced and strom.eqp before installing the drop-in")
    saved = [(red, "ReducedOperator", red.ReducedOperator), (eqp, "ReducedOperator", eqp.ReducedOperator)]
    red.ReducedOperator = GpuReducedOperator
    eqp.ReducedOperator = GpuReducedOperator
    if lm:
        saved.append((eqp, "lm_solve", eqp.lm_solve))
        eqp.lm_solve = gpu_lm_solve

    def undo():
        for mod, name, obj in saved:
            setattr(mod, name, obj)

    return undo
