"""dev check: ghz at several n, both dtypes, direct store on/off (GPU)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2408_09055_b200 import atlas as A
from workloads import circuits as C
for n in (16, 24, 28):
    c = C.ghz(n)
    for d in (0, 1):
        for dt in (0, 1):
            s = A.Simulator(n, dt, 1, 0, shm_direct_store=d)
            s.load_circuit(c.gates); s.plan(); s.run()
            a = s.get_state(0, 1)[0]; b = s.get_state((1 << n) - 1, 1)[0]
            print(n, "direct", d, "dt", dt, a, b, flush=True)
            s.close()
