"""Drop-in installation into the reference package (``rubs``).

The reference binds its engine functions by name at import time in
several modules (pkg/src/rubs/tensor.py:18, cli.py:26, __init__.py:46-53),
so replacing the hot path means patching each of those module attributes.
``install(rubs)`` does exactly that; ``uninstall(rubs)`` restores them.

    import rubs, paper_1003_2022_b200.shim as shim
    shim.install(rubs)            # rubs.filter_space_variant now runs on the B200
    rubs.adaptive_smooth(img, 0.1)  # the reference's own caller, accelerated

Only the filtering path and its own caller, the structure-tensor pipeline
(tensor.py), are replaced; everything else in the reference
(solver, CLI, I/O, oracle) keeps running as shipped.
"""

from __future__ import annotations

import importlib
import sys

from . import engine, tensor

# (module suffix, attribute) -> replacement
_TARGETS = {
    ("engine", "filter_space_variant"): engine.filter_space_variant,
    ("engine", "filter_space_invariant"): engine.filter_space_invariant,
    ("engine", "preintegrate"): engine.preintegrate,
    ("zp", "interpolate"): engine.interpolate,
    ("tensor", "filter_space_variant"): engine.filter_space_variant,
    ("tensor", "filter_space_invariant"): engine.filter_space_invariant,
    ("cli", "filter_space_invariant"): engine.filter_space_invariant,
    ("cli", "filter_space_variant"): engine.filter_space_variant,
    ("", "filter_space_variant"): engine.filter_space_variant,
    ("", "filter_space_invariant"): engine.filter_space_invariant,
    ("", "preintegrate"): engine.preintegrate,
    ("", "interpolate"): engine.interpolate,
    # the reference's own caller of the path (tensor.py), SURVEY.md §8f
    ("tensor", "structure_tensor"): tensor.structure_tensor,
    ("tensor", "anisotropy_from_tensor"): tensor.anisotropy_from_tensor,
    ("tensor", "adaptive_smooth"): tensor.adaptive_smooth,
    ("cli", "adaptive_smooth"): tensor.adaptive_smooth,
    ("", "adaptive_smooth"): tensor.adaptive_smooth,
    ("", "structure_tensor"): tensor.structure_tensor,
}

_SAVED: dict = {}


def _module(pkg, suffix):
    if not suffix:
        return pkg
    name = f"{pkg.__name__}.{suffix}"
    try:
        return sys.modules.get(name) or importlib.import_module(name)
    except ImportError:
        return None


def install(pkg) -> list[str]:
    """Patch the reference package's hot-path bindings; returns what changed."""
    done = []
    for (suffix, attr), fn in _TARGETS.items():
        mod = _module(pkg, suffix)
        if mod is None or not hasattr(mod, attr):
            continue
        key = (mod.__name__, attr)
        if key not in _SAVED:
            _SAVED[key] = getattr(mod, attr)
        setattr(mod, attr, fn)
        done.append(f"{mod.__name__}.{attr}")
    return done


def uninstall(pkg) -> None:
    for (modname, attr), fn in list(_SAVED.items()):
        mod = sys.modules.get(modname)
        if mod is not None:
            setattr(mod, attr, fn)
        del _SAVED[(modname, attr)]
