import sys, os, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2509_01928_b200 as dc
from conftest import golden_k2, k2_W
g = golden_k2()
solver = sys.argv[1] if len(sys.argv) > 1 else "doch"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
inst = dc.ProblemInstance(coupling=dc.maxcut_to_ising(dc.DenseCoupling(k2_W(), validate=False)), cut_offset=595.0)
X0 = np.stack([dc.initial_state(2000, g["alpha"], g["beta"], np.random.default_rng(s)) for s in range(1024)])
res = dc.solve_replicas(inst, solver, g["alpha"], g["beta"], X0, max_iters=iters, precision="f16tc")
res = dc.solve_replicas(inst, solver, g["alpha"], g["beta"], X0, max_iters=iters, precision="f16tc")
print("device s", res[0].device_seconds, "per iter us", 1e6 * res[0].device_seconds / iters)
