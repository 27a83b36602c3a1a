#!/usr/bin/env python
"""bench.py -- Atlas hot path on B200: circuit simulation time and
amplitude-updates/s (BASELINE.json metric), with roofline, CPU-oracle baseline,
end-to-end (host buffers) number and clock record.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload su2random_n28]
                  [--impl reference]

A *step* is one full simulation of the workload circuit through the C-ABI
(atlas_run: |0...0> initialisation, every stage's kernels, every inter-stage
remap).  N=1 runs BASELINE config 2 (su2random, n=28, fp64, one B200).  Under
torchrun with N>1 ranks the run is weak-scaled like the paper's E1 (28 local
qubits per GPU, n = 28 + log2 N) with NCCL remaps between
stages; the timed region is max over ranks.

value   = m * 2^n / T_step  (gate-level amplitude updates per second, SURVEY
          Q24), whole job.
e2e     = same metric through the public API with host buffers: at N = 1
          every step uploads the initial state from pinned host memory, runs,
          and reads the whole final state back (the plan is preprocessing,
          computed once and reported as config.plan.plan_s); at N > 1 every
          step loads the circuit, re-plans, runs and reads one amplitude.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import circuits as C  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)  # >= 4: the autotuning runs
    p.add_argument("--workload", default="su2random_n28")
    p.add_argument("--impl", default="atlas", choices=["atlas", "reference"])
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--kernelizer", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-compare", action="store_true",
                   help="skip re-timing the steps without zero-support tracking (profiling runs)")
    p.add_argument("--opt", action="append", default=[], help="extra library option key=int")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: n = workload n + log2 N (28 local qubits per GPU, the "
                        "paper's E1); strong: n fixed (BASELINE config 4: n = 33 at N = 1/2/4/8)")
    return p.parse_args()


def workload(name, world, scaling="weak"):
    fam, nstr = name.rsplit("_n", 1)
    n = int(nstr)
    if world > 1 and scaling == "weak":
        n += int(math.log2(world))  # weak scaling: 28 local qubits per GPU
    return C.make(fam, n), fam, n


# ---------------------------------------------------------------- clocks
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: wait for its first sample
            # so the timed region that follows is covered
            t_end = time.time() + 5.0
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        self.t0 = time.time()
        self.t1 = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, start: bool):
        """Bracket the timed region (samples outside it are not reported)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        t1 = self.t1 if self.t1 is not None else float("inf")
        # a 100 ms sampler: keep the samples taken inside the timed region
        # (plus one period of slack at the end)
        for t, ln in self.lines:
            if t < self.t0 or t > t1 + 0.1:
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                s = float(f[0])
                mx = float(f[1])
            except ValueError:
                continue
            sm.append(s)
            for name, v in zip(REASONS, f[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"], "samples": 0}
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU oracle
def host_info():
    """nproc, CPU model and RAM of the host the oracle runs on."""
    info = {"nproc": os.cpu_count()}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                info["ram_gb"] = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return info


def cpu_oracle_sample(circ, budget_s=12.0, max_gates=None, omp=True):
    """Time the oracle (as it stands) on the first g gates of the workload at
    full n (g sized to ~budget_s; all of them if they fit).  omp: the OpenMP
    build on every host core, else the 1-thread build.  Returns (updates/s,
    g, seconds)."""
    from oracle import sim as O
    n = circ.n
    # calibrate on one gate (includes the |0> init, so an upper bound)
    t0 = time.perf_counter()
    O.simulate(C.Circuit(n, circ.gates[:1]), omp=omp)
    per_gate = max((time.perf_counter() - t0) * 0.8, 1e-7)
    g = max(1, min(len(circ.gates), int(budget_s / per_gate)))
    if max_gates:
        g = min(g, max_gates)
    t0 = time.perf_counter()
    O.simulate(C.Circuit(n, circ.gates[:g]), omp=omp)
    dt = time.perf_counter() - t0
    return g * (2.0 ** n) / dt, g, dt


def cpu_baseline(fam, n_full, budget_s=10.0):
    """The oracle on the host cores: full circuits of
    the workload's family at n = 12, 20, 24 on 1 core and on all cores
    (n = 24 on 1 core: a leading-gate sample), and the workload itself at
    n_full on all cores as a leading-gate sample (labelled extrapolation:
    rate x whole circuit).  Returns the cpu_baseline object; its value is
    the all-cores rate at the workload size."""
    from oracle import sim as O
    O.build()
    nthr = O.threads(True)
    rows = []
    for n in (12, 20, 24):
        c = C.make(fam, n)
        for omp in (False, True):
            if n == 24 and not omp:
                v, g, dt = cpu_oracle_sample(c, budget_s=budget_s / 2, omp=False)
            else:
                t0 = time.perf_counter()
                O.simulate(c, omp=omp)
                dt = time.perf_counter() - t0
                g = len(c.gates)
                v = g * 2.0 ** n / dt
            rows.append({"n": n, "cores": nthr if omp else 1, "gates": g, "of": len(c.gates),
                         "s": round(dt, 3), "amp_updates_per_s": v,
                         "kind": "full circuit" if g == len(c.gates) else "leading-gate sample"})
    c = C.make(fam, n_full)
    v, g, dt = cpu_oracle_sample(c, budget_s=budget_s, omp=True)
    est = len(c.gates) * 2.0 ** n_full / v
    rows.append({"n": n_full, "cores": nthr, "gates": g, "of": len(c.gates), "s": round(dt, 3),
                 "amp_updates_per_s": v, "kind": "leading-gate sample",
                 "extrapolated_full_circuit_s": round(est, 1)})
    return {"value": v, "unit": "amp-updates/s", "cores": nthr, "kind": "oracle",
            "sample": f"first {g} of {len(c.gates)} gates of {fam} n={n_full} (complex128 "
                      f"gate-at-a-time C oracle, OpenMP over {nthr} host threads, {dt:.1f} s); "
                      f"full circuit extrapolated: {est:.0f} s (labelled extrapolation)",
            "host": host_info(), "by_size": rows}


def load_peaks():
    try:
        d = json.load(open(PEAKS_FILE))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def bench_config(fam, n, m, world, fp64=True):
    """The workload this line measures -- identical for both arms (the
    implementation's own details go to the line's 'details')."""
    amp = 16 if fp64 else 8
    return {"workload": f"{fam}_n{n}_{'fp64' if fp64 else 'fp32'}", "n": n, "gates": m,
            "l2": "state (%.0f GiB/GPU) >> L2; no flush needed" % (amp * 2 ** (n - int(math.log2(world))) / 2 ** 30)}


# ------------------------------------------------------------- reference
def run_reference(args):
    """The tier's reference arm: the oracle as it stands (OpenMP build, every
    host core), each step the leading gates of the workload at full n, sized
    so that warm-up + steps end within ~3 minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    circ, fam, n = workload(args.workload, args.gpus, args.scaling)
    from oracle import sim as O
    O.build()
    nthr = O.threads(True)
    budget = max(0.5, min(6.0, 150.0 / max(1, args.warmup + args.steps)))
    vals = []
    per = None
    for i in range(args.warmup + args.steps):
        v, g, dt = cpu_oracle_sample(circ, budget_s=budget, max_gates=per)
        per = g
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    ms = statistics.median(dt for _, dt in vals) * 1e3
    line = {
        "impl": "reference", "metric": "amplitude-updates/s (circuit simulation)",
        "value": value, "unit": "amp-updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if args.scaling == "weak" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": bench_config(fam, n, len(circ.gates), args.gpus),
        "cpu_baseline": {"value": value, "unit": "amp-updates/s", "cores": nthr, "kind": "oracle",
                         "sample_gates_per_step": per,
                         "sample": f"first {per} of {len(circ.gates)} gates of {fam} n={n} "
                                   f"(complex128, gate-at-a-time C oracle, OpenMP over {nthr} "
                                   f"host threads) per step", "host": host_info()},
        "e2e": {"value": value, "unit": "amp-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------- atlas
def run_atlas(args):
    import numpy as np
    import torch
    from paper_2408_09055_b200 import atlas as A

    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        assert dist.get_world_size() == world
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    circ, fam, n = workload(args.workload, world, args.scaling)
    dtype = A.C128 if args.dtype == "f64" else A.C64
    uid = None
    if world > 1:
        obj = [A.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.Stream()
    extra = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.opt}
    sim = A.Simulator(n, dtype, world, rank, uid, kernelizer=args.kernelizer, device=dev, **extra)
    sim.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    sim.load_circuit(circ.gates)
    sim.plan(16, 3.0)
    plan_s = time.perf_counter() - t0
    stats = sim.plan_stats()
    m = len(circ.gates)
    updates = m * float(2 ** n)

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up (uploads the plan, allocates the shard)
    for _ in range(args.warmup):
        sim.run()
    torch.cuda.synchronize()
    jit_s = sim.plan_stats()["jit_us"] / 1e6  # first run: SHM kernel codegen + NVRTC
    sim.set_option("timing", 1)
    launches = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            sim.run()
            launches.extend(sim.launches())
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    barrier()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = updates / (ms_step / 1e3)
    sim.set_option("timing", 0)

    # the same steps without zero-support tracking (option zero_skip: tiles
    # provably zero in and out are not visited while the run is still inside
    # the support the circuit has reached from |0...0>), so the effect of
    # that exact optimisation on the headline is visible
    no_skip = None
    if extra.get("zero_skip", 1) and not args.no_compare:
        sim.set_option("zero_skip", 0)
        for _ in range(2):
            sim.run()
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            sim.run()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms2 = ev0.elapsed_time(ev1)
        if dist is not None:
            t = torch.tensor([ms2], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms2 = float(t.item())
        no_skip = {"ms_per_step": round(ms2 / args.steps, 4), "value": updates / (ms2 / args.steps / 1e3)}
        sim.set_option("zero_skip", 1)

    # roofline: dominant kernel kind by total device time
    by = {}
    for kind, t, b in launches:
        if kind not in ("fused", "shm", "pack", "scale"):
            continue
        d = by.setdefault(kind, [0.0, 0, 0])
        d[0] += t
        d[1] += 1
        d[2] += b
    step_kernel_ms = sum(v[0] for v in by.values()) / args.steps
    dom = max(by, key=lambda k: by[k][0]) if by else None
    peak, peak_src = load_peaks()
    roof = None
    if dom:
        tot_ms, cnt, byts = by[dom]
        avg_ms = tot_ms / cnt
        bytes_per = byts / cnt
        ach = bytes_per / (avg_ms / 1e3) / 1e9
        traffic = load_traffic().get(f"{dom}_{args.workload}_{args.dtype}")
        roof = {"bound": "hbm", "kernel": f"{dom}_kernel", "achieved": round(ach, 1),
                "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic, "peak_source": peak_src,
                "launches_per_step": cnt / args.steps, "avg_launch_ms": round(avg_ms, 4),
                "share_of_step": round(tot_ms / args.steps / ms_step, 4),
                "bytes_per_launch": int(bytes_per)}
        # the launches that move the full shard (read + write every
        # amplitude): the zero-skip / lazy-zero launches move far fewer bytes
        # while still computing, which lowers the aggregate above
        full_b = 2 * (16 if dtype == A.C128 else 8) * 2 ** (n - int(math.log2(world)))
        dense = [(t, b) for k, t, b in launches if k == dom and b == full_b]
        if dense:
            dt_ = sum(t for t, _ in dense) / len(dense)
            roof["full_pass_launches"] = {
                "per_step": len(dense) / args.steps, "avg_launch_ms": round(dt_, 4),
                "achieved": round(full_b / (dt_ / 1e3) / 1e9, 1),
                "frac": round(full_b / (dt_ / 1e3) / 1e9 / peak, 4)}
    kinds_ms = {k: round(v[0] / args.steps, 4) for k, v in by.items()}
    remap_ms = sum(t for k, t, b in launches if k == "exchange") / args.steps
    # NVLink roofline of the inter-stage all-to-all (north_star): algorithmic
    # bytes each rank sends per remap, (1 - 2^-g') 2^L B, over the measured
    # peer-copy bandwidth per direction (B200_PROFILING.md: 770 GB/s)
    nvlink = None
    xb = sum(b for k, t, b in launches if k == "exchange")
    if world > 1 and xb == 0 and stats["remaps"] > 0:
        # fused exchange (option shm_fuse_exchange): the blocks go to the
        # peers inside the last shared-memory launch of each stage; the
        # remap record only times the closing 4-byte allreduce, so there is
        # no separate exchange time to divide by
        pj_st = sim.plan_json()["stages"]
        amp = 16 if dtype == A.C128 else 8
        sb = sum((1 - 2.0 ** -st["remap_qubits"]) * amp * 2 ** (n - int(math.log2(world)))
                 for st in pj_st if st.get("exchange_fused"))
        nvlink = {"bound": "nvlink", "fused": True, "achieved": None, "peak": 770.0, "unit": "GB/s",
                  "frac": None, "bytes_per_step": int(sb), "remap_ms_per_step": round(remap_ms, 4),
                  "peak_source": "B200_PROFILING.md measured peer copy per direction",
                  "note": "exchange stores ride on the last shared-memory launch of each stage"}
    elif world > 1 and remap_ms > 0:
        ach = (xb / args.steps) / (remap_ms / 1e3) / 1e9  # this rank's bytes / its remap time
        nvlink = {"bound": "nvlink", "achieved": round(ach, 1), "peak": 770.0, "unit": "GB/s",
                  "frac": round(ach / 770.0, 4), "peak_source": "B200_PROFILING.md measured peer copy per direction",
                  "bytes_per_step": int(xb / args.steps), "remap_ms_per_step": round(remap_ms, 4)}
    n_launch = sum(1 for k, t, b in launches if k in ("fused", "shm", "pack", "scale", "init"))

    # e2e: host buffers through the public API.  N = 1: every step uploads
    # the initial state from pinned host memory (atlas_set_state), simulates
    # (atlas_run) and reads the whole final state back into pinned host memory
    # (atlas_get_state); the plan is the circuit's preprocessing (computed
    # once; reported as config.plan.plan_s).  N > 1: every step
    # loads the circuit from host, re-plans, runs and reads one amplitude.
    e2e = None
    if not args.no_e2e:
        amp = 16 if dtype == A.C128 else 8
        reps = max(1, min(3, args.steps))
        barrier()
        if world == 1:
            # two contexts (same circuit, plan = preprocessing) on two
            # streams with option async: step i runs on context i % 2, so the
            # device->host read of one step's result overlaps the
            # host->device upload of the next step's input and the compute
            # (full-duplex PCIe); every step still moves its whole input in
            # and its whole result out
            count = 1 << n
            h_in = torch.zeros(count * amp, dtype=torch.uint8, pin_memory=True)
            h_in[:amp].view(torch.float64 if amp == 16 else torch.float32)[0] = 1.0  # |0...0>
            h_out = [torch.empty(count * amp, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            sim2 = A.Simulator(n, dtype, world, rank, uid, kernelizer=args.kernelizer, device=dev, **extra)
            stream2 = torch.cuda.Stream()
            sim2.set_stream(stream2.cuda_stream)
            sim2.load_circuit(circ.gates)
            sim2.plan(16, 3.0)
            sims, streams = [sim, sim2], [stream, stream2]
            for sm in sims:
                sm.set_option("timing", 0)
                sm.set_option("init", 0)
                sm.set_option("async", 1)
                for _ in range(5 if sm is sim2 else 1):  # warm: JIT + autotuning runs of the second context
                    sm.set_state_from(h_in.data_ptr(), 0, count)
                    sm.run()
            torch.cuda.synchronize()
            reps = max(4, min(8, args.steps))
            t0 = time.perf_counter()
            for i in range(reps):
                j = i % 2
                streams[j].synchronize()  # this context's previous step (and its result read) is done
                sims[j].set_state_from(h_in.data_ptr(), 0, count)
                sims[j].run()
                sims[j].get_state_into(h_out[j].data_ptr(), 0, count)
            for st_ in streams:
                st_.synchronize()
            dt = (time.perf_counter() - t0) / reps
            for sm in sims:
                sm.set_option("async", 0)
                sm.set_option("init", 1)
            sim2.close()
            h2d, d2h = count * amp, count * amp
            inc = ("per step: set_state(full state from pinned host) + run + get_state(full state -> "
                   "pinned host); two contexts on two streams (option async) so consecutive steps overlap "
                   f"their copies and compute; {reps} steps")
        else:
            # N > 1: the plan is preprocessing as at N = 1; every step each
            # rank uploads its logical block [r 2^L, (r+1) 2^L) of the
            # initial state from pinned host memory, runs, and reads its
            # logical block of the result back (atlas_set_state /
            # atlas_get_state fill the entries the rank owns)
            count = 1 << (n - int(math.log2(world)))
            h_in = torch.zeros(count * amp, dtype=torch.uint8, pin_memory=True)
            if rank == 0:
                h_in[:amp].view(torch.float64 if amp == 16 else torch.float32)[0] = 1.0
            h_out = torch.empty(count * amp, dtype=torch.uint8, pin_memory=True)
            sim.set_option("timing", 0)
            sim.set_option("init", 0)
            first = rank * count
            barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                sim.set_state_from(h_in.data_ptr(), first, count)
                sim.run()
                sim.get_state_into(h_out.data_ptr(), first, count)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / reps
            sim.set_option("init", 1)
            h2d, d2h = count * amp, count * amp
            inc = ("per rank: set_state(its logical block from pinned host) + run + "
                   "get_state(its logical block -> pinned host); plan = preprocessing")
        if dist is not None:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": updates / dt, "unit": "amp-updates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 3),
               "includes": inc}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(fam, n)
    sim.close()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    pj = {"stages": stats["stages"], "remaps": stats["remaps"], "kernels": stats["kernels"],
          "fusion_kernels": stats["fusion_kernels"], "shm_kernels": stats["shm_kernels"],
          "plan_s": round(plan_s, 3), "staging_exact": bool(stats["staging_exact"]),
          "shm_jit": bool(extra.get("shm_jit", 1)), "jit_s": round(jit_s, 3)}
    line = {
        "metric": "amplitude-updates/s (circuit simulation)",
        "value": value, "unit": "amp-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "config": bench_config(fam, n, m, world, dtype == A.C128),
        "details": {"L": stats["L"], "G": stats["G"],
                   "parallelism": f"state sharded over {world} GPU(s); remaps fused into the last "
                                  f"shared-memory launch of a stage (peer stores) or NCCL send/recv",
                   "plan": pj, "kernel_ms_per_step": kinds_ms,
                   "remap_ms_per_step": round(remap_ms, 4),
                   "kernels_ms_per_step_total": round(step_kernel_ms, 4),
                   "zero_skip": bool(extra.get("zero_skip", 1)),
                   "zero_skip_note": ("exact, not an approximation: a run from |0...0> does not visit "
                                      "tiles (or store zeros) it proves zero from the qubits no launch "
                                      "has touched yet; without_zero_skip re-times the same steps with "
                                      "zero_skip (and lazy zeros) off"),
                   "without_zero_skip": no_skip},
        "roofline": roof,
        "nvlink": nvlink,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": n_launch,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_atlas(args)


if __name__ == "__main__":
    main()
