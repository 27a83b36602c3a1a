"""Virtual-world timing of the remap paths on one GPU (all W shards on one
device): per-step device time by launch kind with the exchange fused into
the last shared-memory launch of each stage (default) vs the fused pack +
separate exchange copies (shm_fuse_exchange=0) vs standalone packs.

  python tools/virtual_world_bench.py su2random 28 8 [steps]

In a virtual world the 'exchange' is device-to-device copies between the
shards (the NCCL send/recv leg on a multi-GPU box); with the fused exchange
those copies disappear into the stores of the last launch of each stage."""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09055_b200 import atlas as A  # noqa: E402
from workloads import circuits as C  # noqa: E402

fam, L, W = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
n = L + (W.bit_length() - 1)
c = C.make(fam, n)
for name, opts in [("fused exchange", {}), ("fused pack + exchange copies", {"shm_fuse_exchange": 0}),
                   ("standalone pack + exchange copies", {"shm_fuse_exchange": 0, "shm_fuse_pack": 0})]:
    with A.Simulator(n, 0, W, 0, virtual_world=1, **opts) as s:
        s.load_circuit(c.gates)
        s.plan()
        s.run()
        s.run()  # autotune runs
        s.run()
        s.set_option("timing", 1)
        by = defaultdict(float)
        for _ in range(steps):
            s.run()
            for kind, ms, b in s.launches():
                by[kind] += ms / steps
        st = s.plan_stats()
    tot = sum(by.values())
    print(json.dumps({"workload": f"{fam}_n{n}", "W": W, "variant": name, "ms_per_step": round(tot, 3),
                      "by_kind_ms": {k: round(v, 3) for k, v in by.items()},
                      "kernels": st["kernels"], "remaps": st["remaps"]}), flush=True)
