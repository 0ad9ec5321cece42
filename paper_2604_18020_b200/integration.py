"""Binding the B200 kernels into the reference package's own operator.

The reference resolves its kernel module in ``MatFreeOperator.__init__``
(``operator.py:66``: ``self.kernels = get_backend(backend)``), where
``get_backend`` is the name ``operator.py:24`` imported from ``backend.py``
at module import -- so patching ``topofuse.backend.get_backend`` alone does
not reach it, and ``backend.py:42-43`` rejects any name but numpy/numba.
``register_reference_backend`` rebinds the name in BOTH modules (and in the
registry ``_BACKENDS``), leaving every other reference behaviour untouched:

    import topofuse
    from paper_2604_18020_b200.integration import register_reference_backend
    register_reference_backend(topofuse)                  # adds backend="b200"
    op = topofuse.MatFreeOperator(mesh, edof, bcs, rho, backend="b200")
    op.apply(v)        # reference masking/pass-through, B200 fused kernel

``replace="numba"`` instead serves the B200 module under the reference's
default backend name, which is how the reference's own test files run
against it unchanged (``tests/reference_backend_plugin.py``).
``unregister_reference_backend`` restores the original bindings.

Kernel contract (``backend.py:38-46``, ``_kernels_numba.py``): host numpy
arrays in, ``out``/``acc`` accumulated in place -- ``kernels.py``.
"""

from __future__ import annotations

import os

_SAVED = "_b200_saved_bindings"


def _modules(topofuse=None):
    if topofuse is None:
        import topofuse
    import importlib

    tb = importlib.import_module(topofuse.__name__ + ".backend")
    top = importlib.import_module(topofuse.__name__ + ".operator")
    return topofuse, tb, top


def register_reference_backend(topofuse=None, name: str = "b200", replace: str | None = None):
    """Make the reference's MatFreeOperator resolve ``name`` (or, with
    ``replace``, an existing backend name) to the B200 kernel module.
    Returns that module.  Idempotent; undo with unregister_reference_backend."""
    from . import kernels

    topofuse, tb, top = _modules(topofuse)
    if not hasattr(tb, _SAVED):
        setattr(tb, _SAVED, (tb.get_backend, top.get_backend, dict(tb._BACKENDS)))
    orig = getattr(tb, _SAVED)[0]
    served = replace or name
    tb._BACKENDS[served] = kernels

    def get_backend(backend: str | None = None):
        # same resolution order as backend.py:38-46: explicit, env, default
        key = backend
        if key is None:
            key = os.environ.get(tb.ENV_VAR, "").strip().lower() or tb.default_backend_name()
        if key == served:
            return kernels
        return orig(backend)

    get_backend.__doc__ = orig.__doc__
    tb.get_backend = get_backend
    top.get_backend = get_backend  # the binding operator.py:66 actually calls
    return kernels


def unregister_reference_backend(topofuse=None) -> None:
    topofuse, tb, top = _modules(topofuse)
    saved = getattr(tb, _SAVED, None)
    if saved is None:
        return
    tb.get_backend, top.get_backend, regs = saved
    tb._BACKENDS.clear()
    tb._BACKENDS.update(regs)
    delattr(tb, _SAVED)
