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


# BASELINE.json configs the bench times (SURVEY.md §8 size table):
# name -> (preset, scale).  Inputs follow the reference bench convention
# (bench.py:161-173): rho ~ U(0.05, 1) then v ~ N(0, 1) from default_rng(42).
BASELINE_CASES = {
    "c3": ("torsion", 1.0),
    "c4": ("cantilever", 5 / 3),
    "c5": ("cantilever", 17 / 6),
}


def baseline_case(name):
    """(mesh, edof, bcs, rho, v) of a BASELINE config, as
    tests/golden/make_golden_r2.py drew them for the reference."""
    from paper_2604_18020_b200.mesh import build_edof, make_preset

    preset, scale = BASELINE_CASES[name]
    pb = make_preset(preset, scale)
    m = pb.mesh
    rng = np.random.default_rng(42)
    rho = rng.uniform(0.05, 1.0, m.n_elem)
    v = rng.standard_normal(m.n_dof)
    return m, build_edof(m), pb.bcs, rho, v


def sample_index(n, k=4097):
    """Entries sampled by make_golden_r2.py (4097 evenly spaced DOFs)."""
    return np.unique(np.linspace(0, n - 1, k).astype(np.int64))
