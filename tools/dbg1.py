import sys, numpy as np
sys.path.insert(0,'/root/repo')
from paper_2408_09055_b200 import atlas as A
from workloads import circuits as C
from oracle import sim as O
c=C.su2random(13)
ref=O.simulate(c)
for d in (0,1):
    s=A.Simulator(13,0,1,0,shm_direct=d); s.load_circuit(c.gates); s.plan(); s.run(); psi=s.get_state()
    print("direct",d,"maxdiff",np.abs(psi-ref).max(), flush=True)
    s.close()
