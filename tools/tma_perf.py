"""A/B wall-clock per run (atlas's own stream; each run ends with a stream
sync) -- debugging aid for the TMA loads."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09055_b200 import atlas as A
from workloads import circuits as C

fam, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
for variant in sys.argv[4:]:
    opts = {} if variant == "-" else {kv.split("=")[0]: int(kv.split("=")[1]) for kv in variant.split(",")}
    c = C.make(fam, n)
    with A.Simulator(n, 0, 1, 0, **opts) as s:
        s.load_circuit(c.gates)
        s.plan()
        for _ in range(3):
            s.run()
        t0 = time.perf_counter()
        for _ in range(reps):
            s.run()
        dt = (time.perf_counter() - t0) / reps
    print(f"{fam} n={n} {variant}: {dt * 1e3:.3f} ms/run", flush=True)
