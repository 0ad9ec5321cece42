"""CPU-side tests: host mirror of the reference API, C-ABI library exports,
and the no-fallback guarantee.  No kernel is launched here."""

from __future__ import annotations

import ctypes
import hashlib
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_available, load_golden
from paper_2604_18020_b200 import _lib
from paper_2604_18020_b200.element import SimpParams, simp_scale, unit_stiffness
from paper_2604_18020_b200.mesh import (CORNER_OFFSETS, StructuredMesh, build_edof,
                                        cantilever_bcs, edof_is_structured, make_preset)


def test_library_exports_every_header_symbol():
    import os

    # RTLD_NOW: every symbol the library needs must resolve at load (catches a
    # template used across translation units but defined with internal linkage)
    L = ctypes.CDLL(str(_lib.LIB_PATH), mode=os.RTLD_NOW)
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert _lib.load().tf_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(cuda_available(), reason="checks the GPU-less failure mode")
def test_operator_fails_loudly_without_gpu():
    from paper_2604_18020_b200 import MatFreeOperator

    m = StructuredMesh(2, 2, 2)
    with pytest.raises(_lib.TfError):
        MatFreeOperator(m, build_edof(m), cantilever_bcs(m), np.full(m.n_elem, 0.5))


def test_unit_stiffness_matches_reference_golden():
    ke = unit_stiffness(0.3)
    ref = load_golden("ke.npz")["ke"]
    # bitwise: the exact-order kernels and the Jacobi diagonal consume these bits
    assert np.array_equal(ke, ref)
    assert np.array_equal(ke.astype(np.float32), ref.astype(np.float32))
    assert np.array_equal(ke, ke.T)
    w = np.linalg.eigvalsh(ke)
    assert int((np.abs(w) <= 1e-9 * np.abs(w).max()).sum()) == 6


def test_edof_matches_reference_hashes():
    h = load_golden("hashes.json")
    for dims in [(4, 3, 2), (24, 12, 6), (48, 24, 24), (120, 60, 30)]:
        e = build_edof(StructuredMesh(*dims))
        assert hashlib.sha256(e.tobytes()).hexdigest() == h["edof_" + "x".join(map(str, dims))]


def test_structured_detection():
    m = StructuredMesh(5, 4, 3)
    e = build_edof(m)
    assert edof_is_structured(m, e)
    e2 = e.copy()
    e2[7, 3] += 3
    assert not edof_is_structured(m, e2)
    assert not edof_is_structured(m, e[:-1])


def test_presets_and_bcs():
    pb = make_preset("cantilever", 0.2)
    assert (pb.mesh.nelx, pb.mesh.nely, pb.mesh.nelz) == (24, 12, 6)
    assert pb.bcs.fixed_dofs.size == 3 * 13 * 7
    assert pb.bcs.force.sum() == -1.0
    t = make_preset("torsion", 0.2)
    assert abs(t.bcs.force.sum()) < 1e-15
    with pytest.raises(ValueError):
        make_preset("cantilever", 0.123)
    with pytest.raises(ValueError):
        StructuredMesh(0, 1, 1)
    assert CORNER_OFFSETS.shape == (8, 3)


def test_simp_scale_and_validation():
    assert np.allclose(simp_scale(np.array([0.0, 1.0])), [1e-9, 1.0])
    with pytest.raises(ValueError):
        simp_scale(np.array([1.5]))
    with pytest.raises(ValueError):
        SimpParams(p=0.5)


def test_filter_oc_schedule_host_logic():
    from paper_2604_18020_b200.simp import (build_cone_filter, default_schedule,
                                            heaviside_projection, oc_update)

    m = StructuredMesh(5, 5, 5)
    w = build_cone_filter(m, 1.5).toarray()
    c = m.element_id(2, 2, 2)
    z = 1.5 + 6 * 0.5 + 12 * (1.5 - np.sqrt(2.0))
    assert abs(w[c, c] - 1.5 / z) < 1e-13 and (w[c] > 0).sum() == 19
    assert np.allclose(w.sum(axis=1), 1.0)
    e = heaviside_projection(np.array([0.0, 0.5, 1.0]), 16.0)
    assert np.allclose(e, [0.0, 0.5, 1.0], atol=1e-15)
    rng = np.random.default_rng(17)
    rho = rng.uniform(0.05, 0.95, 128)
    new = oc_update(rho, -rng.uniform(0.1, 10, 128), np.ones(128), 0.4, move=0.2)
    assert abs(new.mean() - 0.4) <= 1e-6
    s = default_schedule(120)
    assert s.at(1).p == 1.5 and s.at(120).beta == 32.0


def test_filter_matches_reference_construction():
    """Same CSR values as the reference's filter on a small mesh (bitwise rows)."""
    from paper_2604_18020_b200.simp import build_cone_filter

    m = StructuredMesh(4, 3, 2)
    got = build_cone_filter(m, 1.5).toarray()
    # O(n^2) restatement of the cone weights (reference tests/oracles.py:161-175)
    cen = m.element_centers()
    d = np.sqrt(((cen[:, None, :] - cen[None, :, :]) ** 2).sum(-1))
    W = np.maximum(0.0, 1.5 - d)
    assert np.max(np.abs(got - W / W.sum(1, keepdims=True))) <= 1e-14


def test_traffic_model_numbers():
    from paper_2604_18020_b200.operator import compulsory_bytes, traffic_model

    assert traffic_model("fused", "fp32").bytes_with_indices == 292
    assert traffic_model("three_stage", "fp64").bytes_with_indices == 868
    assert compulsory_bytes(216000, 686433, "fp32", False) == 216000 * 100 + 8 * 686433


def test_density_snapshot_roundtrip_and_reference_layout(tmp_path):
    from paper_2604_18020_b200.snapshot import read_density, write_density

    rho = np.random.default_rng(2).uniform(0, 1, 4 * 3 * 2)
    b, j = write_density(tmp_path / "d", rho, (4, 3, 2))
    assert b.read_bytes() == rho.astype("<f8").tobytes()
    import json as _json

    assert _json.loads(j.read_text()) == {"count": 24, "dims": [4, 3, 2], "dtype": "float64",
                                          "order": "x-fastest"}
    got, dims = read_density(tmp_path / "d")
    assert dims == (4, 3, 2) and np.array_equal(got, rho)
    with pytest.raises(ValueError):
        write_density(tmp_path / "e", rho[:-1], (4, 3, 2))


def test_node_fixed_layout_host_restatement():
    from paper_2604_18020_b200._device import node_fixed_mask

    m = StructuredMesh(3, 2, 2)
    bcs = cantilever_bcs(m)
    nf = node_fixed_mask(m.n_nodes, bcs.fixed_dofs, (m.nelx + 1) * (m.nely + 1))
    pn = (m.nelx + 1) * (m.nely + 1)
    assert nf.size == m.n_nodes + 2 * pn
    col_or, col_and = nf[m.n_nodes:m.n_nodes + pn], nf[m.n_nodes + pn:]
    # clamped x=0 face: all three bits on every plane -> z-invariant
    for j in range(m.nely + 1):
        assert col_or[j * (m.nelx + 1)] == 7 and col_and[j * (m.nelx + 1)] == 7
    assert col_or[1] == 0


def test_simp_artifacts_byte_identical_to_reference(tmp_path):
    """History CSV, summary JSON and selected-density snapshot written for a
    fixed synthetic result are byte-identical to the reference's cmd_simp
    output for the same result (tests/golden/make_golden_artifacts.py)."""
    import sys

    from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset
    from paper_2604_18020_b200 import simp as S
    from paper_2604_18020_b200.snapshot import write_simp_artifacts

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_golden_artifacts import synthetic_result

    pb = make_preset("cantilever", 0.1)
    cfg = SimpConfig(schedule=default_schedule(6))
    res = synthetic_result(S, pb, cfg)
    paths = write_simp_artifacts(tmp_path, res, pb, "fp64", "fused", "serial", iters=6, cg_cap=1000, seed=42)
    gold = Path(__file__).resolve().parent / "golden" / "artifacts"
    names = {p.name for p in gold.iterdir()}
    assert names == {"simp_cantilever_fp64_history.csv", "simp_cantilever_fp64_summary.json",
                     "simp_cantilever_fp64_selected.bin", "simp_cantilever_fp64_selected.json"}
    for name in names:
        assert (tmp_path / name).read_bytes() == (gold / name).read_bytes(), name
    assert paths["history"].name == "simp_cantilever_fp64_history.csv"


def test_ctypes_struct_layouts_match_the_c_abi():
    """The ctypes mirrors of the public structs have the C compiler's sizes
    (a field added on one side only would shift every later field)."""
    L = _lib.load()
    out = (ctypes.c_int64 * 5)()
    assert L.tf_abi_struct_sizes(out, 5) == 0
    mirrors = [_lib.tf_grid, _lib.tf_pcg_desc, _lib.tf_pcg_report, _lib.tf_oc_report, _lib.tf_slab_desc]
    assert [ctypes.sizeof(m) for m in mirrors] == list(out)


def test_id_cache_releases_entries_with_their_key():
    """cached values must not pin their key; the entry goes when
    the key object dies (a value holding only a weakref)."""
    import gc
    import weakref

    from paper_2604_18020_b200._device import IdCache

    c = IdCache()

    class Val:
        def __init__(self, key):
            self.ref = weakref.ref(key)

    keys = [np.zeros(4) for _ in range(5)]
    for k in keys:
        c.get(k, "x", lambda k=k: Val(k))
    assert len(c) == 5
    del k
    keys.clear()
    gc.collect()
    assert len(c) == 0


def test_constraint_digest_is_content_keyed():
    """id(bcs) is reused by CPython; the device-problem key is the
    constraint content."""
    from paper_2604_18020_b200.mesh import BoundaryConditions
    from paper_2604_18020_b200.operator import _constraint_digest

    m = StructuredMesh(3, 2, 2)
    digests = set()
    for k in range(6):
        b = BoundaryConditions(np.arange(k, k + 3, dtype=np.int64), np.zeros(m.n_dof))
        digests.add(_constraint_digest(b))
        del b
    assert len(digests) == 6
    b1 = BoundaryConditions(np.array([1, 2, 3]), np.zeros(m.n_dof))
    b2 = BoundaryConditions(np.array([1, 2, 3]), np.ones(m.n_dof))
    assert _constraint_digest(b1) == _constraint_digest(b2)


def test_device_glue_only_for_structured_fused_configs():
    """bf16 and grid_kernel='edof' keep the host glue (run_simp
    chooses, the device loop would refuse them)."""
    import inspect

    from paper_2604_18020_b200 import simp

    src = inspect.getsource(simp.run_simp)
    assert 'grid_kernel != "edof"' in src and '"bf16"' in src
