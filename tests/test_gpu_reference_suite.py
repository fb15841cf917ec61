"""GPU: the reference's OWN hot-path tests, run against the drop-in.

The unmodified reference (dcising 0.1.0, pip-installed into baseline/_ref with
its test directory beside it; git-ignored, shipped to the GPU box) is copied to
a temporary directory and patched exactly as INTEGRATION.md §1 tells a
maintainer to: an import override at the end of ``dcising/solvers/__init__.py``
routes ``doch_solve`` / ``adoch_solve`` / ``apply_T`` / ``hamiltonian`` /
``hamiltonian_gradient`` to paper_2509_01928_b200 (libdcx.so on the B200).
Then the reference's pytest suite runs in a subprocess on that copy:

* ``pkg/tests/test_doch.py`` in full (fixed points, descent inequality, step
  decay :177-185, boundedness, residuals after convergence :229-236, best of
  restarts :238-249, time budget, ADOCH replay and the paired ADOCH-vs-DOCH
  comparison :366-376, ...);
* acceptance criteria 1-3, 5, 6 and 12 (``pkg/tests/test_acceptance.py:51-200,
  344-372``): monotone descent, boundedness, fixed-point convergence, tiny-scale
  optimality, the two-spin figure, the gradient check.

A first test file written next to them asserts that the override is active, so
the suite cannot pass on the reference's own numpy loop by accident.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not (REF / "dcising").is_dir() or not (REF / "tests").is_dir(),
                       reason="baseline/_ref (reference install + its tests) not present"),
]

PATCH = '''

# --- B200 drop-in (INTEGRATION.md section 1) ---------------------------------
try:
    from paper_2509_01928_b200 import (adoch_solve, apply_T, doch_solve, hamiltonian,  # noqa: F401
                                       hamiltonian_gradient)
except ImportError:
    pass
'''

ACTIVE = '''
import dcising.solvers as s


def test_drop_in_is_active():
    for name in ("doch_solve", "adoch_solve", "apply_T", "hamiltonian", "hamiltonian_gradient"):
        assert getattr(s, name).__module__.startswith("paper_2509_01928_b200"), name
    r = s.doch_solve(__import__("dcising").ProblemInstance(coupling=__import__("dcising").DenseCoupling(
        __import__("numpy").array([[0.0, -1.0], [-1.0, 0.0]]))), __import__("dcising").SolverParams(alpha=1.0, beta=2.0))
    assert r.path in ("persistent", "multipass")  # ran through libdcx.so
'''

ACCEPTANCE = ["test_criterion_01_monotone_descent", "test_criterion_02_boundedness_rule",
              "test_criterion_03_fixed_point_convergence", "test_criterion_05_tiny_scale_optimality",
              "test_criterion_06_two_spin_reproduction", "test_criterion_12_gradient_check"]


def test_reference_hot_path_suite_through_drop_in(tmp_path):
    src = tmp_path / "src"
    shutil.copytree(REF / "dcising", src / "dcising")
    with open(src / "dcising" / "solvers" / "__init__.py", "a") as f:
        f.write(PATCH)
    shutil.copytree(REF / "tests", tmp_path / "tests")
    (tmp_path / "tests" / "test_00_drop_in_active.py").write_text(ACTIVE)
    env = dict(os.environ, PYTHONPATH=f"{src}{os.pathsep}{ROOT}", PYTHONWARNINGS="ignore::RuntimeWarning")
    sel = ["tests/test_00_drop_in_active.py", "tests/test_doch.py"] + \
          [f"tests/test_acceptance.py::{t}" for t in ACCEPTANCE]
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x", *sel],
                          cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join((proc.stdout + proc.stderr).splitlines()[-40:])
    assert proc.returncode == 0, tail
    assert " passed" in proc.stdout and "failed" not in proc.stdout, tail
