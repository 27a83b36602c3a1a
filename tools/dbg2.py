import sys, numpy as np
sys.path.insert(0,'/root/repo')
from paper_2408_09055_b200 import atlas as A
from workloads import circuits as C
for n in (16, 20, 24, 26, 28):
    c=C.ghz(n)
    for d in (0,1):
        for dt in (0,1):
            s=A.Simulator(n,dt,1,0,shm_direct=d); s.load_circuit(c.gates); s.plan(); s.run()
            a=s.get_state(0,1)[0]; b=s.get_state((1<<n)-1,1)[0]
            pj=s.plan_json()
            ks=[(k['kind'],k['qubits'],k['gates']) for st in pj['stages'] for k in st['kernels']]
            print(n,"direct",d,"dt",dt,a,b, "K", pj['K_tile'], flush=True)
            if abs(b)<0.5: print(ks)
            s.close()
