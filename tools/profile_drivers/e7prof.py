import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2509_01928_b200 as dc
from paper_2509_01928_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "e7"
it = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if name == "e7":
    n = 10**7; v, c, o, co = synth.erdos_renyi(n, 8, seed=0, device=0); alpha, beta = 2.828, 5.005e11
else:
    n = 10**8; v, c, o, co = synth.random_regular3(n, seed=0, device=0); alpha, beta = 1.732, 3.232e12
inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False), cut_offset=co)
X0 = dc.initial_state(n, alpha, beta, np.random.default_rng(0))[None, :]
for rep in range(2):
    r = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=it, precision="f32", path="multipass")
    print(name, "device ms/iter", 1e3 * r[0].device_seconds / it, flush=True)
