"""Host planner (C++ in libatlas_b200.so, through the C-ABI) against the
oracle planners -- bit-exact where the oracle is exact (staging optimum with
its canonical tie-break, OrderedKernelize), bounds + validity for Kernelize.
CPU only: atlas_create/load/plan make no CUDA call."""
import json
import os

import pytest

from oracle import gates as OG, planner as P
from workloads import circuits as C

A = pytest.importorskip("paper_2408_09055_b200.atlas")
try:
    A.lib()
except Exception as e:  # pragma: no cover
    pytest.skip(f"library not built: {e}", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))


def test_library_exports_every_header_symbol():
    """include/atlas.h declares exactly the exported C entry points."""
    import re
    hdr = open(os.path.join(HERE, "..", "include", "atlas.h")).read()
    declared = set(re.findall(r"\b(atlas_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(A.SYMBOLS), declared ^ set(A.SYMBOLS)
    lib = A.lib()
    for s in declared:
        assert hasattr(lib, s), s


def test_errors_are_status_codes():
    with pytest.raises(A.AtlasError) as e:
        A.Simulator(10, world=3)
    assert e.value.status == 1
    s = A.Simulator(4)
    with pytest.raises(A.AtlasError) as e:
        s.load_circuit([C.Gate("CX", (0, 5))])
    assert e.value.status == 1
    with pytest.raises(A.AtlasError) as e:
        s.run()  # before plan
    assert e.value.status == 8
    with pytest.raises(A.AtlasError) as e:
        s.set_option("no_such_option", 1)
    assert e.value.status == 2
    # a gate with more non-insular qubits than L is infeasible
    s = A.Simulator(3, world=4, virtual_world=1)
    s.load_circuit([C.Gate("SWAP", (0, 1)), C.Gate("H", (2,))])
    with pytest.raises(A.AtlasError) as e:
        s.plan()
    assert e.value.status == 3


def product_plan(c, world, **opt):
    s = A.Simulator(c.n, world=world, virtual_world=1 if world > 1 else 0, **opt)
    s.load_circuit(c.gates)
    s.plan(8, 3.0)
    return s.plan_json()


def masks(qs):
    return sorted(qs)


# ------------------------------------------------------------------ staging
STAGING_CASES = [(C.ghz(3), 2), (C.qft(6), 8), (C.qft(5), 4), (C.ghz(6), 4)]
STAGING_CASES += [(C.random_circuit(5, 9, 40 + s, kinds=("H", "X", "Z", "CX", "CZ", "CP", "RY", "T"),
                                    max_arity=2), (2, 4, 8)[s % 3]) for s in range(10)]


@pytest.mark.parametrize("case", range(len(STAGING_CASES)))
def test_staging_matches_bruteforce(case):
    """Minimum s (Thm. ilp-optimal), minimum objective (Eq. P:L1477)
    and the canonical tie-break must equal the brute-force oracle bit for bit."""
    c, world = STAGING_CASES[case]
    G = world.bit_length() - 1
    L = c.n - G
    bf = P.stage_bruteforce(c, L=L, Gq=G, s_max=4, c=3)
    pj = product_plan(c, world)
    st = pj["staging"]
    assert st["s"] == bf.s
    assert st["cost"] == pytest.approx(bf.cost)
    assert st["gate_stage"] == bf.gate_stage
    for k in range(bf.s):
        assert pj["stages"][k]["global"] == masks(bf.globals[k])
        assert pj["stages"][k]["local"] == masks(bf.locals[k])


def test_staging_c_invariance():
    """With R = 0 the plan does not depend on c and J = (1 + c) * swaps
    (reading R7; BASELINE config 5's c sweep)."""
    c = C.qft(8)
    plans = []
    for cf in (1.0, 2.0, 3.0, 5.0, 10.0):
        s = A.Simulator(8, world=4, virtual_world=1)
        s.load_circuit(c.gates)
        s.plan(8, cf)
        pj = s.plan_json()
        plans.append([st["global"] for st in pj["stages"]])
        swaps = sum(len(set(pj["stages"][k]["global"]) - set(pj["stages"][k - 1]["global"]))
                    for k in range(1, pj["staging"]["s"]))
        assert pj["staging"]["cost"] == pytest.approx((1 + cf) * swaps)
    assert all(p == plans[0] for p in plans)


# ----------------------------------------------------------- kernelization
def model_json(tmp_path, qmf=4, qms=6, ls=0, alpha=300, fus=(100, 110, 150, 400)):
    d = {"fusion_cost": list(fus[:qmf]), "alpha": alpha,
         "gate_cost": {k: {1: 20, 2: 30, 3: 40}[C.ARITY[k]] for k in C.KINDS},
         "q_max_fusion": qmf, "q_max_shared": qms, "ls_qubits": ls}
    p = tmp_path / "cm.json"
    p.write_text(json.dumps(d))
    return str(p), P.CostModel.from_json(d)


def oracle_seq(c):
    """Kernelizer input by the oracle's own insularity: active = operands that
    are not diagonal-type (reading R16: anti-diagonal local qubits are active)."""
    out = []
    for g in c.gates:
        ins = OG.insular_kind(g.kind, g.params)
        out.append(P.KGate(frozenset(g.qubits),
                           frozenset(q for q, t in zip(g.qubits, ins) if t != "diag"),
                           g.kind))
    return out


@pytest.mark.parametrize("seed", range(12))
def test_ordered_kernelize_matches_bruteforce(tmp_path, seed):
    """OrderedKernelize == min over all contiguous segmentations,
    with the same segments (canonical tie-break R21) and kinds."""
    n = 7
    c = C.random_circuit(n, 11, 600 + seed, kinds=("H", "X", "CX", "CZ", "CP", "RZ", "U3", "SWAP", "CCX"))
    path, cm = model_json(tmp_path, ls=seed % 3)
    pj = product_plan(c, 1, kernelizer=1, cost_model=path)
    seq = oracle_seq(c)
    ls = frozenset(range(seed % 3))
    cost, segs = P.ordered_bruteforce(seq, cm, ls, n)
    ks = pj["stages"][0]["kernels"]
    assert pj["stages"][0]["kernel_cost"] == cost
    assert [k["gates"] for k in ks] == [list(range(a, b)) for a, b, _ in segs]
    assert [k["kind"] for k in ks] == [kd for _, _, kd in segs]


@pytest.mark.parametrize("fam", ["qft", "ghz", "su2random", "ising", "qsvm", "wstate", "graphstate"])
@pytest.mark.parametrize("lift", [0, 1])
def test_kernelize_valid_and_not_worse_than_ordered(tmp_path, fam, lift):
    """Thm. dp-correct: the kernels concatenate to a sequence
    topologically equivalent to the stage; Thm. dp-optimal: cost
    <= OrderedKernelize."""
    n = 9
    c = C.make(fam, n)
    path, cm = model_json(tmp_path, qms=7, ls=2)
    pj = product_plan(c, 1, kernelizer=0, cost_model=path, insular_lift=lift)
    po = product_plan(c, 1, kernelizer=1, cost_model=path)
    seq = oracle_seq(c)
    ks = pj["stages"][0]["kernels"]
    errs, cost = P.verify_plan([k["gates"] for k in ks], [k["kind"] for k in ks], seq, cm,
                               frozenset(range(2)), n, lift=True, check_constraint1=False)
    assert errs == []
    assert cost == pj["stages"][0]["kernel_cost"]
    assert cost <= po["stages"][0]["kernel_cost"]


@pytest.mark.parametrize("seed", range(6))
def test_kernelize_bounded_by_bruteforce(tmp_path, seed):
    """BF_opt <= Kernelize (plain Constraint 1: no lifting, no attachment)."""
    n = 5
    c = C.random_circuit(n, 6, 800 + seed, kinds=("H", "CX", "CZ", "U3", "RZ"), max_arity=2)
    path, cm = model_json(tmp_path, qms=6, qmf=4)
    pj = product_plan(c, 1, kernelizer=0, cost_model=path, insular_lift=0, attach=0)
    seq = oracle_seq(c)
    bf, _ = P.kernel_bruteforce(seq, cm, frozenset(), n)
    assert bf <= pj["stages"][0]["kernel_cost"]
    ks = pj["stages"][0]["kernels"]
    for k in ks:
        assert P.satisfies_constraint1(set(k["gates"]), [g.qubits for g in seq])


def test_kernelize_beats_ordered_on_su2random():
    """The non-contiguous DP must find plans OrderedKernelize cannot
    (App. P:L2390-2394, Fig. dp-pruning)."""
    c = C.su2random(14)
    pk = product_plan(c, 1, kernelizer=0, shm_qubits=8)
    po = product_plan(c, 1, kernelizer=1, shm_qubits=8)
    assert pk["stages"][0]["kernel_cost"] < 0.8 * po["stages"][0]["kernel_cost"]


def test_greedy_baseline_is_fusion_up_to_5(tmp_path):
    c = C.qft(10)
    pj = product_plan(c, 1, kernelizer=2)
    for k in pj["stages"][0]["kernels"]:
        assert k["kind"] == "fusion" and len(k["qubits"]) <= 5


@pytest.mark.parametrize("fam", ["qft", "su2random", "ising", "qsvm", "wstate", "random"])
def test_front_packing_valid(tmp_path, fam):
    """The front packing (R29) yields kernels whose concatenation is
    topologically equivalent to the stage (checked by the oracle's
    verify_plan, Thm. dp-correct's notion) and whose reported cost
    is the model cost of those kernels."""
    n = 9
    c = C.random_circuit(n, 40, 901, kinds=("H", "X", "CX", "CZ", "CP", "RZ", "U3", "SWAP", "CCX")) \
        if fam == "random" else C.make(fam, n)
    path, cm = model_json(tmp_path, qms=7, ls=2)
    pj = product_plan(c, 1, kernelizer=3, cost_model=path)
    seq = oracle_seq(c)
    ks = pj["stages"][0]["kernels"]
    errs, cost = P.verify_plan([k["gates"] for k in ks], [k["kind"] for k in ks], seq, cm,
                               frozenset(range(2)), n, lift=True, check_constraint1=False)
    assert errs == []
    assert cost == pj["stages"][0]["kernel_cost"]


def test_front_packing_cx_block_windows():
    """An all-to-all CX block (su2random's entangler) needs one kernel per
    window of q_max_shared - ls target qubits across all rows: 20 qubits, 2^12
    tiles with 5 forced LSB qubits -> targets 1..11, 12..18, 19: 3 kernels."""
    from workloads.circuits import Gate, Circuit
    n = 20
    c = Circuit(n, [Gate("CX", (i, j)) for i in range(n) for j in range(i + 1, n)])
    pj = product_plan(c, 1, kernelizer=3, kinds=2, ls_qubits=5)
    assert len(pj["stages"][0]["kernels"]) == 3
    pk = product_plan(c, 1, kernelizer=0, kinds=2, ls_qubits=5)
    assert len(pk["stages"][0]["kernels"]) == 3
    # ls_auto (ls_qubits unset): 4 forced LSB qubits -> windows of 8 targets
    # (4..11, 12..19) -> 2 kernels; the model keeps the cheaper plan
    pa = product_plan(c, 1, kernelizer=3, kinds=2)
    assert pa["ls_qubits"] in (4, 5)
    assert len(pa["stages"][0]["kernels"]) <= 3


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("W", [2, 4, 8])
def test_exchange_is_pairwise_swap_up_to_flip_relabel(seed, W):
    """The property the in-place remap (option inplace_remap, NEXT-3) relies
    on: in every remap, each rank sends to peer p the block at offset o and
    receives p's block at o XOR (incoming flips, as a block index) -- the
    same relabelling for every peer and for the block that stays local -- and
    p does the mirror image.  So a pairwise in-place block swap followed by
    one xor relabel pass reproduces the out-of-place exchange exactly."""
    n = 10
    c = C.random_circuit(n, 60, 500 + seed, kinds=("H", "X", "Y", "CX", "CZ", "RZ", "U3", "SWAP"),
                         max_arity=2)
    scheds = []
    for r in range(W):
        with A.Simulator(n, 0, W, r) as s:
            s.load_circuit(c.gates)
            s.plan()
            S = s.plan_json()["staging"]["s"]
            scheds.append({k: s.remap_schedule(k) for k in range(1, S)})
    for k in scheds[0]:
        for r in range(W):
            xs = scheds[r][k]
            if not xs:
                continue
            sends = {x[1]: x[2] for x in xs if x[0] == "send"}
            recvs = {x[1]: x[3] for x in xs if x[0] == "recv"}
            local = [x for x in xs if x[0] == "local"]
            assert len(local) == 1 and set(sends) == set(recvs)
            rel = local[0][2] ^ local[0][3]  # the flip relabel of this remap (bytes)
            for p, so in sends.items():
                assert recvs[p] ^ so == rel
                # the peer's pair of transfers with us has the same shape
                psend = {x[1]: x[2] for x in scheds[p][k] if x[0] == "send"}
                prec = {x[1]: x[3] for x in scheds[p][k] if x[0] == "recv"}
                assert prec[r] ^ psend[r] == rel


def test_fused_pack_present():
    """su2random at W = 8 needs packs; with fusion every one of them rides
    on a shared-memory launch (no standalone pack launch).  Host-only: the
    plan report."""
    c = C.su2random(20)
    with A.Simulator(c.n, 0, 8, 0, virtual_world=1) as s:
        s.load_circuit(c.gates)
        s.plan()
        pj = s.plan_json()
    packed = [st for st in pj["stages"] if st["packed"]]
    assert packed and all(st["pack_fused"] for st in packed)


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("fam", ["su2random", "qft", "ising"])
def test_exchange_fused_plan(fam, W):
    """shm_fuse_exchange: every remap's exchange rides on the previous
    stage's last shared-memory launch (packed remaps and, with an identity
    pack, unpacked ones); off, none does.  Host-only: the plan report."""
    c = C.make(fam, 20)
    for on in (1, 0):
        with A.Simulator(c.n, 0, W, 0, virtual_world=1, shm_fuse_exchange=on) as s:
            s.load_circuit(c.gates)
            s.plan()
            pj = s.plan_json()
        remaps = [st for st in pj["stages"][1:] if st["remap_qubits"] > 0]
        assert remaps
        assert all(bool(st["exchange_fused"]) == bool(on) for st in remaps)


@pytest.mark.parametrize("key", ["async", "zero_skip", "init", "timing", "shm_addr_split", "shm_fold_perm",
                                 "shm_lit_smem", "shm_tma"])
def test_runtime_options_keep_the_plan(key):
    """Options that only change how a plan runs (not the plan) can be set
    between atlas_plan and atlas_run: the plan stays valid (host-only)."""
    c = C.su2random(14)
    with A.Simulator(c.n, 0, 1, 0) as s:
        s.load_circuit(c.gates)
        s.plan()
        before = s.plan_json()
        s.set_option(key, 1)
        s.set_option(key, 0)
        assert s.plan_json() == before
        assert s.jit_source(0)
