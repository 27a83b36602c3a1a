"""The plan-specialised shared-memory kernels (csrc/jit.cpp, R30) on the CPU
box: atlas_get_jit_source is host-only, so the generated CUDA is checked
here without a GPU -- it compiles for sm_100a with nvcc (the same compiler
front end NVRTC uses on the GPU box), stays within the register budget of
its launch bounds without spilling, and reflects the lowered program
(phases, zero-mode initialisation, the pipelined variant).  GPU parity of
the same kernels is in test_gpu_parity.py."""
import os
import re
import shutil
import subprocess

import pytest

from workloads import circuits as C

A = pytest.importorskip("paper_2408_09055_b200.atlas")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
pytestmark = pytest.mark.skipif(not (os.path.exists(NVCC) or shutil.which("nvcc")),
                                reason="nvcc not available")


def sources(circ, dtype=0, **opt):
    out = []
    with A.Simulator(circ.n, dtype, 1, 0, **opt) as s:
        s.load_circuit(circ.gates)
        s.plan()
        n_shm = s.plan_stats()["shm_kernels"]
        for i in range(n_shm):
            out.append(s.jit_source(i))
        with pytest.raises(A.AtlasError):
            s.jit_source(n_shm)
    return out


def ptxas(src, tmp_path, name):
    cu = tmp_path / f"{name}.cu"
    cu.write_text(src)
    r = subprocess.run([NVCC, "-cubin", "-arch=sm_100a", "-std=c++17", "-Xptxas", "-v",
                        str(cu), "-o", str(tmp_path / f"{name}.cubin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    regs = int(re.search(r"Used (\d+) registers", r.stderr).group(1))
    spill = re.search(r"(\d+) bytes spill stores", r.stderr)
    return regs, int(spill.group(1)) if spill else 0


@pytest.mark.parametrize("fam,dtype", [("su2random", 0), ("qsvm", 0), ("ising", 0), ("qft", 1),
                                       ("su2random", 1), ("random", 0)])
def test_jit_sources_compile_without_spills(fam, dtype, tmp_path):
    """Every launch of the plan compiles within its launch bounds.  The
    benchmark families (the kernels bench.py times) must not spill at all.
    The all-kinds random circuit may spill a few words: its conditional
    register permutations (X/CX/SWAP with thread/tile-dependent controls
    that cannot be folded into addresses, OP_PERM1) keep two copies of 16
    complex doubles live at the 128-register cap of the 512-thread pipe CTA;
    it is a parity workload, not a bench one."""
    c = C.random_circuit(16, 160, 17) if fam == "random" else C.make(fam, 16)
    srcs = sources(c, dtype)
    assert srcs, "plan has no shared-memory kernel"
    for i, src in enumerate(srcs):
        m = re.search(r"__launch_bounds__\((\d+), (\d+)\)", src)
        threads, minb = int(m.group(1)), int(m.group(2))
        regs, spill = ptxas(src, tmp_path, f"k{i}")
        assert regs * threads * minb <= 65536
        assert spill <= (64 if fam == "random" else 0), f"kernel {i} spills {spill} bytes"


def test_jit_source_reflects_program():
    """One source per shared-memory launch; the header names K, RB and the
    phase count of the lowered program; the first launch of a run from
    |0...0> can synthesise its input (zmode) in the single-buffer pipeline."""
    c = C.su2random(16)
    srcs = sources(c)
    assert "#define ZERO_OK 1" in srcs[0]
    for src in srcs:
        assert re.search(r"K=\d+ RB=\d+ phases=\d+ ops=\d+", src)
        # a kernel whose leading permutation-only phase is folded into the
        # load cannot synthesise |0...0> in that phase (never a first launch
        # of a run from |0...0> in these plans)
        if "folded into the tile load" in src:
            assert "#define ZERO_OK 0" in src
            continue
        assert "#define ZERO_OK 1" in src
        assert "(zmode & 3) == 2 && tile == 0 && jt == 0" in src
        # zero tiles of a zmode launch: stored as zeros, no phases (linearity;
        # a shared-memory kernel keeps every tile inside itself)
        assert "if (zmode && ((zmode & 3) == 1 || tile != 0)) {" in src
        # shared-memory addresses: one pointer per distinct low (bank) part
        assert re.search(r"T \*q\d+ = tb \+ \(sj \^ \d+\);", src)
    # plan-specialised: no op-program interpretation in the generated code
    assert "switch" not in srcs[0]


@pytest.mark.parametrize("fam", ["su2random", "qsvm"])
@pytest.mark.parametrize("pipe", [0, 1])
def test_jit_pipe_variant_compiles(fam, pipe, tmp_path):
    """Both pipelines on every launch: pipe mode (one CTA of two groups, six
    mbarriers: tile i completes on barrier i % 6) and the two-CTA single
    buffer (cp.async groups)."""
    c = C.make(fam, 16)
    srcs = sources(c, shm_pipe=pipe)
    for i, src in enumerate(srcs):
        assert ("mbarrier.try_wait.parity" in src) == bool(pipe)
        if pipe:
            assert "for (int i = 0; i < 6; i++)" in src and "mbar_wait(mbar0 + 8 * mb, (i / 6) & 1)" in src
        m = re.search(r"__launch_bounds__\((\d+), (\d+)\)", src)
        regs, spill = ptxas(src, tmp_path, f"p{i}")
        assert regs * int(m.group(1)) * int(m.group(2)) <= 65536 and spill == 0


def test_fold_leading_permutation_phase():
    """A leading phase that only carries a folded permutation (su2random's
    CX block before the next U3 layer) is folded into the tile load: the
    kernel says so, cannot synthesise |0...0> (ZERO_OK 0) and emits one
    phase fewer; with shm_fold_perm = 0 the phase is emitted."""
    c = C.su2random(28)
    on = sources(c)
    off = sources(c, shm_fold_perm=0)
    folded = [i for i, src in enumerate(on) if "folded into the tile load" in src]
    assert folded, "no kernel folded its leading permutation phase"
    for i in folded:
        assert "#define ZERO_OK 0" in on[i]
        assert on[i].count("{ // phase ") == off[i].count("{ // phase ") - 1


def test_fused_exchange_kernels_compile(tmp_path):
    """The last shared-memory launch of each stage of a W = 8 plan carries
    the exchange (ATLAS_PEER: stores into the destination ranks' blocks);
    it compiles for sm_100a without spills and picks its destination block
    from the shared-memory table once per tile (no per-store local-memory
    pointer load)."""
    c = C.su2random(20)
    with A.Simulator(c.n, 0, 8, 0, virtual_world=1) as s:
        s.load_circuit(c.gates)
        s.plan()
        srcs = [s.jit_source(i, 3) for i in range(s.plan_stats()["shm_kernels"])]
    peer = [src for src in srcs if "#define ATLAS_PEER" in src]
    assert peer
    for i, src in enumerate(peer):
        assert "ptab_s[" in src and "ptab.p[threadIdx.x]" in src
        regs, spill = ptxas(src, tmp_path, f"x{i}")
        assert spill == 0
