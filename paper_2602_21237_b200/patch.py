"""Install the B200 operators into a live ``relab`` package.

The reference binds the tensor-path functions by name at import time
(bench.py:49 ``from .tensorpath import ... tensor_join, tensor_sort,
to_tensor``; the package re-exports them, __init__.py:60-67), so a drop-in
must rebind the names in every module that holds them. After ``install()``
the unmodified reference harness (``run_experiment``, the CLI, the tests)
runs its tensor path on the B200 kernels and sees relab's own record and
exception classes. ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib

from . import tensor_path as _tp

OPERATORS = ("to_tensor", "key_axis_align", "tensor_join", "tensor_sort")
CLASSES = ("TensorRelation", "AxisAlignment")
_saved: dict = {}


def _modules():
    names = ("relab", "relab.tensorpath", "relab.bench")
    return [importlib.import_module(n) for n in names]


def install() -> list:
    """Rebind relab's tensor-path names to this package. Returns the
    (module, name) pairs that were replaced."""
    errors = importlib.import_module("relab.errors")
    spill = importlib.import_module("relab.spill")
    _saved.setdefault("TYPES", dict(_tp.TYPES))
    _tp.TYPES.update(
        SpillStats=spill.SpillStats,
        OutputTooLarge=errors.OutputTooLarge,
        UnknownAttribute=errors.UnknownAttribute,
    )
    replaced = []
    for mod in _modules():
        for name in OPERATORS + CLASSES:
            if hasattr(mod, name):
                _saved.setdefault((mod.__name__, name), getattr(mod, name))
                setattr(mod, name, getattr(_tp, name))
                replaced.append((mod.__name__, name))
    return replaced


def uninstall() -> None:
    for key, value in list(_saved.items()):
        if key == "TYPES":
            _tp.TYPES.clear()
            _tp.TYPES.update(value)
            continue
        modname, name = key
        setattr(importlib.import_module(modname), name, value)
    _saved.clear()
