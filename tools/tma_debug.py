"""Small-n TMA / pipeline smoke on the GPU (each case under its own timeout
in tools/gpu_tma_debug.sh): max |d| against the oracle."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_09055_b200 import atlas as A
from oracle import sim as O
from workloads import circuits as C

fam, n = sys.argv[1], int(sys.argv[2])
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[3:]}
reps = opts.pop("reps", 1)
c = C.make(fam, n)
with A.Simulator(n, 0, 1, 0, **opts) as s:
    s.load_circuit(c.gates)
    s.plan()
    for r in range(reps):
        s.run()
        print("run", r, "a0", s.get_state(0, 1)[0], flush=True)
    psi = s.get_state()
if n <= 24:
    ref = O.simulate(c)
    print(fam, n, opts, "max|d| = %.3e" % np.abs(psi - ref).max(), flush=True)
else:
    print(fam, n, opts, "ran; norm = %.12f" % np.linalg.norm(psi), flush=True)
