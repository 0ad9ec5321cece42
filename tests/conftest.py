"""Shared test setup: markers, repo path, golden-fixture helpers."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name: str):
    p = GOLDEN / name
    if p.suffix == ".json":
        return json.loads(p.read_text())
    return np.load(p, allow_pickle=False)


@pytest.fixture(scope="session")
def golden_ke():
    return load_golden("ke.npz")["ke"]


def seeded_case(dims, seed):
    """Inputs exactly as tests/golden/make_golden.py:matvec_case draws them."""
    from paper_2604_18020_b200.mesh import StructuredMesh, build_edof, cantilever_bcs

    m = StructuredMesh(*dims)
    edof = build_edof(m)
    bcs = cantilever_bcs(m)
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.05, 1.0, m.n_elem)
    v = rng.standard_normal(m.n_dof)
    return m, edof, bcs, rho, v


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
