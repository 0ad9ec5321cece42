"""paper_2604_18020_b200 -- B200-native matrix-free Q1-hex K.v + Jacobi-PCG.

Drop-in for the hot path of the reference ``topofuse`` package: the same
public names for mesh/BC setup, the matrix-free operator, the CG solvers,
sensitivities, OC update and the SIMP driver, with every evaluation running
in hand-written sm_100a kernels (libtopofuse_b200.so) on the current CUDA
device.  There is no CPU fallback.
"""

from .element import (RHO_MIN, SimpParams, assemble_dense, elasticity_matrix, simp_scale,
                      simp_scale_derivative, unit_stiffness)
from .mesh import (DESK_SCALE, PRESET_NAMES, BoundaryConditions, ProblemPreset, StructuredMesh,
                   build_edof, cantilever_bcs, edof_is_structured, make_preset)
from .operator import (DEVICE_CEILINGS, FLOPS_PER_ELEMENT, SCATTER_MODES, VARIANTS,
                       MatFreeOperator, RooflineConfig, TrafficReport, compulsory_bytes,
                       effective_bandwidth, jacobi_diagonal, memory_footprint, roofline_bound,
                       traffic_model)
from .precision import (BF16, EPS_BF16, EPS_FP32, EPS_FP64, FP32, FP64, Precision, get_precision,
                        quantize, round_to_bf16)
from .simp import (ContinuationSchedule, Phase, SimpConfig, SimpResult, build_cone_filter,
                   chain_to_design, compliance_sensitivity, default_schedule, grayness,
                   heaviside_derivative, heaviside_projection, oc_update, run_simp)
from .solver import (CgConfig, DivergenceError, IrConfig, IrReport, SolveReport, device_pcg,
                     fp64_relative_residual, pcg, solve_equilibrium, solve_refined)

__version__ = "0.1.0"


def available_backends() -> tuple[str, ...]:
    return ("b200",)


def default_backend_name() -> str:
    return "b200"


def get_backend(name: str | None = None):
    """Kernel module for the reference contract (backend.py:38-46)."""
    if name not in (None, "b200"):
        raise ValueError(f"unknown backend {name!r}, expected b200")
    from . import kernels

    return kernels
