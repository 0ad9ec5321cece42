"""Reference-side binding mechanics (no GPU needed): the B200 kernel module
is reached from the REFERENCE's own MatFreeOperator (operator.py:24,66) and
INTEGRATION.md's snippet runs verbatim.  Skipped when the reference package
is not importable (the GPU box has it only as baseline/_ref)."""

from __future__ import annotations

import re
import sys

import numpy as np
import pytest

from conftest import ROOT, cuda_available


def reference_path():
    for p in (ROOT / "baseline" / "_ref", ROOT.parent / "reference" / "pkg" / "src"):
        if (p / "topofuse" / "operator.py").exists():
            return p
    return None


@pytest.fixture
def topofuse():
    p = reference_path()
    if p is None:
        pytest.skip("reference package not importable here")
    sys.path.insert(0, str(p))
    try:
        import topofuse as tf
    except Exception as e:  # numba missing etc.
        pytest.skip(f"reference import failed: {e!r}")
    from paper_2604_18020_b200.integration import unregister_reference_backend

    yield tf
    unregister_reference_backend(tf)
    sys.path.remove(str(p))


def test_registered_backend_reaches_b200_kernels(topofuse):
    import paper_2604_18020_b200.kernels as b200
    from paper_2604_18020_b200 import _lib
    from paper_2604_18020_b200.integration import register_reference_backend

    with pytest.raises(ValueError):  # backend.py:42-43 before registration
        topofuse.MatFreeOperator(*_small(topofuse), backend="b200")
    register_reference_backend(topofuse)
    op = topofuse.MatFreeOperator(*_small(topofuse), backend="b200")
    assert op.kernels is b200
    # the reference's default and explicit names are untouched
    assert topofuse.MatFreeOperator(*_small(topofuse)).kernels is not b200
    assert topofuse.backend.get_backend("numpy").__name__.endswith("_kernels_numpy")
    v = np.random.default_rng(0).standard_normal(op.n_dof)
    if not cuda_available():
        # the call crossed into the B200 package: it fails loudly (no CPU fallback)
        with pytest.raises(_lib.TfError):
            op.apply(v)


def test_replace_default_name_and_unregister(topofuse):
    import paper_2604_18020_b200.kernels as b200
    from paper_2604_18020_b200.integration import register_reference_backend, unregister_reference_backend

    register_reference_backend(topofuse, replace="numba")
    assert topofuse.MatFreeOperator(*_small(topofuse), backend="numba").kernels is b200
    assert "numba" in topofuse.backend.available_backends()
    unregister_reference_backend(topofuse)
    assert topofuse.MatFreeOperator(*_small(topofuse), backend="numba").kernels is not b200


def test_integration_md_snippet_runs_verbatim(topofuse):
    """INTEGRATION.md §2's code block, executed as written."""
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text.split("## 2.")[1].split("## 3.")[0]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    import paper_2604_18020_b200.kernels as b200

    assert ns["op"].kernels is b200


def _small(tf):
    m = tf.StructuredMesh(4, 3, 2)
    rho = np.random.default_rng(11).uniform(0.05, 1.0, m.n_elem)
    return m, tf.build_edof(m), tf.cantilever_bcs(m), rho
