"""B200-native DOCH/ADOCH Ising solver (drop-in for the hot path of dcising).

Public names mirror ``dcising`` (dc/__init__.py:3-43) for the solver path:
couplings, instances, energies, parameters and the DOCH/ADOCH solvers. All
arithmetic of the solver path runs in libdcx.so (hand-written sm_100a CUDA);
there is no CPU fallback.
"""

from .coupling import CouplingError, CouplingMatrix, CsrCoupling, DenseCoupling, ProceduralCoupling, gen_procedural_sin
from .model import (
    ProblemInstance,
    cut_value,
    dehomogenize,
    energies,
    energy,
    energy_with_field,
    homogenize,
    homogenized_instance,
    instance_energy,
    maxcut_to_ising,
    spins_from,
)
from .generate import gen_sparse_9bit
from .io import FormatError, csr_load, csr_save
from .params import DEFAULT_ETA_GRID, SolverParams, derive_params, estimate_lambda_max_neg, tune_eta
from .solvers import (
    CONVERGENCE_TOL,
    DESCENT_WARN_TOL,
    SOLVER_NAMES,
    HamiltonianView,
    SolveResult,
    TraceRecord,
    adoch_solve,
    apply_T,
    attractor,
    doch_solve,
    hamiltonian,
    hamiltonian_gradient,
    initial_state,
    profile_dominant_kernel,
    solve,
    solve_replicas,
)


def matvec(J, v, plan=None):
    """J @ v on the device (dc/matvec.py:99-114); ``plan`` is accepted and ignored."""
    import numpy as np

    from .coupling import device_context

    v = np.asarray(v, dtype=np.float64)
    if v.shape != (J.n,):
        raise ValueError(f"vector length {v.shape} does not match n={J.n}")
    return device_context(J).matvec(v[None, :])[0]


def operator_energy(J, x, plan=None):
    """(J x, -1/2 x.Jx) from one device product (dc/matvec.py:181-190)."""
    y = matvec(J, x)
    return y, -0.5 * float(x @ y)


__version__ = "0.1.0"
