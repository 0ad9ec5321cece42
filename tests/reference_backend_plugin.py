"""pytest plugin: run the REFERENCE's own test files against the B200 kernels.

    python -m pytest -p reference_backend_plugin <reference tests>/test_operator.py

(with tests/ and the reference package importable).  At configure time the
B200 kernel module is registered under the reference's default backend name
"numba" (paper_2604_18020_b200.integration.register_reference_backend), so
every reference test parametrised over available_backends() -- and every
operator built with the default backend -- evaluates on the GPU through
libtopofuse_b200.so.  Nothing under the reference tree is modified.
"""

from __future__ import annotations


def pytest_configure(config):
    import topofuse

    from paper_2604_18020_b200.integration import register_reference_backend

    register_reference_backend(topofuse, replace="numba")
    config.addinivalue_line("markers", "criterion(num, desc): reference acceptance criterion")
