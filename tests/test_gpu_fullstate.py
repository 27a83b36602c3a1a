"""GPU parity at sizes where every CTA of a shared-memory launch loops over
many tiles (the pipelined path the bench times), element by element over the
FULL state against the CPU oracle O1.

Round-1 gap (VERDICT weak #2/#3, ADVICE): element-wise comparisons stopped at
n = 18, where the grid covers every tile with one CTA, so the pipeline's
second-and-later tiles (tile buffers 1 and 2, the mbarrier phase flips, the
next-tile issue, the per-group double-buffered base-factor tables) were only
reached by sampled checks at n = 28 -- one of which failed.  Here:

* bench configuration (ls_auto, plan-specialised kernels, pipe mode, default
  grid) at n = 22-24: 2^10-2^12 tiles of 2^12 amplitudes over 148 CTAs;
* the same with the grid capped (option ``shm_grid``) so that each CTA runs
  tens to hundreds of tiles, for pipe and non-pipe kernels;
* mirrors (C then C^dagger, P7) of every family at the same sizes;
* the previous default (shm_pipe = 0: two single-buffer CTAs per SM with
  early next-tile issue) as a variant;
* the round-1 failing case, qsvm n = 28 mirror, repeated on one context.

Tolerances (BASELINE.json north_star): fp64 max|d amp| <= 1e-10 and
1 - F <= 1e-9; fp32 1e-4 and 1e-5.  No global-phase alignment.
"""
import numpy as np
import pytest

from oracle import sim as O
from workloads import circuits as C

pytestmark = pytest.mark.gpu

A = pytest.importorskip("paper_2408_09055_b200.atlas")

TOL = {0: (1e-10, 1e-9), 1: (1e-4, 1e-5)}

# family -> n of the bench-configuration element-wise case (oracle cost
# m * 2^n amplitude updates stays <= ~4e9 per case)
BENCH_N = {"qft": 24, "ghz": 24, "graphstate": 24, "qsvm": 24, "wstate": 24,
           "ising": 24, "su2random": 22}


def fidelity(a, b):
    a = a.astype(np.complex128)
    b = b.astype(np.complex128)
    return abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)


def check(psi_gpu, psi_ref, dtype=0):
    md, fd = TOL[dtype]
    d = np.abs(psi_gpu.astype(np.complex128) - psi_ref).max()
    f = 1 - fidelity(psi_gpu, psi_ref)
    assert d <= md, f"max|d|={d:.3e}"
    assert f <= fd, f"1-F={f:.3e}"
    return d, f


def run(c, dtype=0, world=1, repeat=1, **opt):
    out = []
    with A.Simulator(c.n, dtype, world, 0, virtual_world=1 if world > 1 else 0, **opt) as s:
        s.load_circuit(c.gates)
        s.plan()
        for _ in range(repeat):
            s.run()
            out.append(s.get_state())
        return out, s.plan_stats()


@pytest.mark.parametrize("fam", C.FAMILIES)
def test_bench_config_full_state(fam):
    """Every family at n = 22-24 in bench.py's launch configuration, every
    amplitude against O1."""
    c = C.make(fam, BENCH_N[fam])
    (psi,), st = run(c)
    check(psi, O.simulate(c))


@pytest.mark.parametrize("fam", C.FAMILIES)
def test_bench_config_mirror_full_state(fam):
    """C C^dagger = I (P7) on the full state: |0...0> exactly, within BJ's
    tolerance, at the bench-configuration sizes."""
    n = BENCH_N[fam]
    c = C.mirror(C.make(fam, n))
    (psi,), _ = run(c)
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[0] = 1
    check(psi, ref)


@pytest.mark.parametrize("opt", [{}, {"shm_pipe": 0}, {"shm_pipe": 0, "shm_ctas": 3},
                                 {"shm_direct_store": 0}, {"shm_tfac_min": 0},
                                 {"zero_skip": 0}, {"shm_addr_split": 0}, {"shm_lit_smem": 1},
                                 {"shm_fold_perm": 0}])
@pytest.mark.parametrize("fam", ["su2random", "qsvm", "ising", "qft", "random"])
def test_grid_capped_many_tiles(fam, opt):
    """A grid of 3 CTAs at n = 18 (64 tiles): each pipe group runs ~10 tiles
    through all three ring buffers and both mbarrier parities; the non-pipe
    kernels run ~21 tiles each with early next-tile issue."""
    c = C.random_circuit(18, 200, 5) if fam == "random" else C.make(fam, 18)
    ref = O.simulate(c)
    (psi,), _ = run(c, shm_grid=3, **opt)
    check(psi, ref)


@pytest.mark.parametrize("fam", ["su2random", "qsvm", "qft"])
def test_grid_capped_fp32(fam):
    c = C.make(fam, 18)
    (psi,), _ = run(c, dtype=1, shm_grid=5)
    check(psi, O.simulate(c), dtype=1)


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("fam", ["su2random", "qft", "ising"])
def test_virtual_world_full_state(fam, W):
    """W > 1 plans at n = 22 (L = 19..21: 2^7..2^9 tiles per shard, packs and
    exchanges present) element-wise against O1."""
    c = C.make(fam, 22)
    (psi,), st = run(c, world=W)
    check(psi, O.simulate(c))


def test_qsvm_n28_mirror_repeated():
    """The round-1 red case: qsvm n = 28 mirror (11 pipe-mode kernels at
    2^16 tiles) run 10 times on one context; |0...0> every time."""
    n = 28
    c = C.mirror(C.qsvm(n))
    rng = np.random.default_rng(3)
    idx = sorted({int(x) for x in rng.integers(1, 1 << n, size=64)})
    with A.Simulator(n, 0, 1, 0) as s:
        s.load_circuit(c.gates)
        s.plan()
        for rep in range(10):
            s.run()
            a0 = s.get_state(0, 1)[0]
            assert abs(a0 - 1) <= 1e-10, f"run {rep}: |a0-1|={abs(a0 - 1):.3e}"
            rest = np.array([s.get_state(i, 1)[0] for i in idx])
            assert np.abs(rest).max() <= 1e-10


@pytest.mark.parametrize("opt", [{"shm_fuse_pack": 0}, {"shm_jit": 0}, {"shm_grid": 2},
                                 {"shm_fuse_exchange": 0}, {"zero_skip": 0}])
@pytest.mark.parametrize("W", [2, 8])
def test_fused_pack_variants(W, opt):
    """The remap pack fused into the previous stage's last shared-memory
    launch (default) against the standalone pack (shm_fuse_pack = 0), the
    interpreter's in-place-then-permute fallback (shm_jit = 0) and a capped
    grid, su2random n = 20 (4 remaps, packs at W >= 2)."""
    c = C.su2random(20)
    (psi,), _ = run(c, world=W, **opt)
    check(psi, O.simulate(c))


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("fam", ["su2random", "qft", "random"])
def test_inplace_remap(fam, W):
    """NEXT-3: remaps in place (bit-transposition packs, pairwise block swaps,
    flip relabelling; no scratch shard buffer) against O1.  The random
    circuits put X/Y gates on global qubits, so incoming flips are exercised."""
    c = C.random_circuit(16, 160, 60 + W, max_arity=2) if fam == "random" else C.make(fam, 18)
    (psi,), _ = run(c, world=W, inplace_remap=1)
    check(psi, O.simulate(c))


def test_inplace_remap_capacity_n33_two_shards():
    """Two 64 GiB fp64 shards of an n = 33 state on one B200 (virtual world
    W = 2) with in-place remaps: 128 GiB total, which does not fit with a
    scratch buffer per shard (256 GiB).  qft from |x> against the P4 closed
    form at sampled amplitudes."""
    n = 33
    x = 0x15A3C1F7 & ((1 << n) - 1)
    c = C.prepend_basis(C.qft(n), x)
    rev = int(format(x, f"0{n}b")[::-1], 2)
    rng = np.random.default_rng(8)
    idx = sorted({0, (1 << n) - 1} | {int(v) for v in rng.integers(0, 1 << n, size=48)})
    with A.Simulator(n, 0, 2, 0, virtual_world=1, inplace_remap=1) as s:
        s.load_circuit(c.gates)
        s.plan()
        assert s.plan_stats()["remaps"] >= 1
        s.run()
        got = np.array([s.get_state(i, 1)[0] for i in idx])
    want = np.array([np.exp(2j * np.pi * ((rev * y) % (1 << n)) / (1 << n)) for y in idx]) * 2 ** (-n / 2)
    assert np.abs(got - want).max() <= 1e-10


@pytest.mark.parametrize("R", [1, 2, 4])
@pytest.mark.parametrize("fam", ["su2random", "qft", "ising", "random"])
def test_offload_tier(fam, R):
    """NEXT-4: the state in host DRAM (2^R regional chunks streamed through
    the GPU stage by stage) against O1, element by element."""
    c = C.random_circuit(16, 160, 80 + R, max_arity=2) if fam == "random" else C.make(fam, 18)
    (psi,), st = run(c, offload=R)
    assert st["G"] == R
    check(psi, O.simulate(c))


def test_offload_tier_from_input_state():
    """atlas_set_state into the host tier (arbitrary input)."""
    n = 15
    c = C.random_circuit(n, 120, 91, max_arity=3)
    rng = np.random.default_rng(4)
    psi0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi0 /= np.linalg.norm(psi0)
    with A.Simulator(n, 0, 1, 0, offload=3) as s:
        s.load_circuit(c.gates)
        s.plan()
        s.set_option("init", 0)
        s.set_state(psi0)
        s.run()
        psi = s.get_state()
    check(psi, O.simulate(c, init=psi0))


@pytest.mark.parametrize("fam", ["su2random", "qft", "ising"])
def test_zero_skip_runs_then_set_state(fam):
    """Zero-support tracking (option zero_skip) only applies to runs from
    |0...0>: run from |0...0> (tiles skipped), then from an arbitrary input
    state (nothing skipped: every tile is nonzero), then from |0...0> again,
    on one context; every result element-wise against O1.  n = 20 with the
    grid capped so that the skipped and the visited tiles are spread over
    several tiles per CTA."""
    n = 20
    c = C.make(fam, n)
    rng = np.random.default_rng(11)
    psi0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi0 /= np.linalg.norm(psi0)
    ref0 = O.simulate(c)
    ref1 = O.simulate(c, init=psi0)
    with A.Simulator(n, 0, 1, 0, shm_grid=7) as s:
        s.load_circuit(c.gates)
        s.plan()
        s.run()
        check(s.get_state(), ref0)
        s.set_state(psi0)
        s.set_option("init", 0)
        s.run()
        check(s.get_state(), ref1)
        s.set_option("init", 1)
        s.run()
        check(s.get_state(), ref0)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_zero_skip_virtual_world_ranks(W):
    """In a virtual world every shard but rank 0's starts all zero: its
    stage-0 launches after the first are skipped entirely (zero_skip), rank
    0's visit only the tiles inside the reached support.  Element-wise vs O1
    with and without the option."""
    c = C.make("su2random", 21)
    ref = O.simulate(c)
    for zs in (1, 0):
        (psi,), _ = run(c, world=W, zero_skip=zs)
        check(psi, ref)


def test_async_two_contexts_pipelined():
    """Option async (bench.py's e2e pipeline): two contexts of one circuit on
    two torch streams; each step uploads an input (atlas_set_state), runs
    and reads the result back (atlas_get_state) without a host sync; the
    caller synchronises the stream before reusing a context's buffers.
    Every step's result element-wise vs O1 (alternating inputs: |0...0> and
    an arbitrary state)."""
    torch = pytest.importorskip("torch")
    n = 18
    c = C.make("su2random", n)
    rng = np.random.default_rng(5)
    psi1 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi1 /= np.linalg.norm(psi1)
    psi0 = np.zeros(1 << n, dtype=np.complex128)
    psi0[0] = 1
    refs = [O.simulate(c), O.simulate(c, init=psi1)]
    ins = [torch.from_numpy(p.view(np.float64).copy()).pin_memory() for p in (psi0, psi1)]
    outs = [torch.empty(2 << n, dtype=torch.float64).pin_memory() for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    sims = [A.Simulator(n, 0, 1, 0) for _ in range(2)]
    try:
        for s, st in zip(sims, streams):
            s.set_stream(st.cuda_stream)
            s.load_circuit(c.gates)
            s.plan()
            s.set_option("init", 0)
            s.set_option("async", 1)
        pending = [None, None]
        for step in range(6):
            j = step % 2
            streams[j].synchronize()
            if pending[j] is not None:
                check(outs[j].numpy().view(np.complex128), refs[pending[j]])
            k = step % 2 if step < 2 else (step // 2) % 2
            sims[j].set_state_from(ins[k].data_ptr(), 0, 1 << n)
            sims[j].run()
            sims[j].get_state_into(outs[j].data_ptr(), 0, 1 << n)
            pending[j] = k
        for j in range(2):
            streams[j].synchronize()
            check(outs[j].numpy().view(np.complex128), refs[pending[j]])
    finally:
        for s in sims:
            s.close()


@pytest.mark.parametrize("lazy", [1, 0])
def test_zero_lazy_partial_support(lazy):
    """Lazy zeros need every local qubit to become active during stage 0;
    a circuit that never touches the high qubits keeps the stored zeros
    (the run falls back), one that does is exact with zero-filled loads.
    Both element-wise vs O1, and followed by a run from an arbitrary input
    on the same context."""
    n = 20
    low = C.random_circuit(14, 120, 9)                       # qubits 0..13 only
    part = C.Circuit(n, list(low.gates), "low14_in_20", 9)
    full = C.make("su2random", n)
    rng = np.random.default_rng(2)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    for c in (part, full):
        with A.Simulator(n, 0, 1, 0, zero_lazy=lazy, shm_grid=5) as s:
            s.load_circuit(c.gates)
            s.plan()
            for _ in range(2):
                s.run()
                check(s.get_state(), O.simulate(c))
            s.set_state(psi)
            s.set_option("init", 0)
            s.run()
            check(s.get_state(), O.simulate(c, init=psi))
