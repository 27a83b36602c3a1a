"""Repeated runs of one plan on a torch stream (bench.py's setup); prints
how many runs completed (debugging aid for the TMA pipeline)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import torch
from paper_2408_09055_b200 import atlas as A
from workloads import circuits as C

fam, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[4:]}
use_stream = opts.pop("stream", 1)
torch.cuda.set_device(0)
c = C.make(fam, n)
s = A.Simulator(n, 0, 1, 0, device=0, **opts)
if use_stream:
    st = torch.cuda.Stream()
    s.set_stream(st.cuda_stream)
s.load_circuit(c.gates)
s.plan()
done = 0
try:
    for r in range(reps):
        t0 = time.perf_counter()
        try:
            s.run()
        finally:
            dt = time.perf_counter() - t0
            if dt > 1.0:
                print(f"run {r}: {dt:.2f} s", flush=True)
        done += 1
finally:
    print(fam, n, opts, "stream" if use_stream else "default", "runs completed:", done, "of", reps, flush=True)
