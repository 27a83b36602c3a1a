/*
 * atlas.h -- C-ABI of the B200-native Atlas hot path (arXiv 2408.09055).
 *
 * The library simulates a quantum circuit on a 2^n complex state vector that
 * is sharded over `world` B200 GPUs (one process per GPU), following the
 * paper's problem statement
 *     Simulate(C, state, L, R, G)          PAPER.md P:L1321-1324 (Alg. 1)
 *     = Execute(Partition(C, L, R, G), state)
 * with the physical-qubit hierarchy collapsed onto one 8xB200 NVSwitch box:
 * L = n - log2(world) local qubits (each GPU's HBM shard, Def. P:L1405-1417),
 * R = 0 regional qubits, G = log2(world) global qubits (the rank bits).
 *
 *   atlas_create       Simulate's machine parameters (n, L, R=0, G)
 *   atlas_load_circuit C, a gate sequence
 *   atlas_plan         Partition: Stage (ILP) + Kernelize per
 *                      stage (App. P:L2348-2499) + lowering
 *   atlas_run          Execute: per stage, Shard (remap
 *                      all-to-all) then LaunchKernel for each kernel
 *   atlas_get_state    read amplitudes back in logical order
 *
 * Conventions:
 *  - Amplitude index: logical qubit q is bit q of the index (Eq. 2).
 *  - Gate operands: q[0] is the least-significant bit of the gate's matrix
 *    index.  Controlled kinds list controls first: CX(c,t), CP(c,t), CU(c,t),
 *    CCX(c0,c1,t).  Matrices are the textbook / OpenQASM ones (R2).
 *  - Amplitudes are interleaved (re, im): double2 for ATLAS_C128, float2 for
 *    ATLAS_C64, little endian.
 *
 * Ownership: the context owns the plan and (unless atlas_bind_buffers is
 * used) all device memory.  Gate arrays and host buffers are caller-owned
 * and only read/written during the call.  No call retains a caller pointer
 * except atlas_bind_buffers / atlas_set_stream (borrowed until destroy or
 * rebinding).
 *
 * Errors: every call returns an atlas_status; no exception crosses the ABI.
 * atlas_last_error() returns a thread-local message for the last failure.
 * Device work only starts in atlas_run / atlas_get_state / atlas_set_state;
 * create/load/plan are host-only (usable without a GPU for planning).
 *
 * Threading: a context is not thread-safe; use one context per thread.
 */
#ifndef ATLAS_H_
#define ATLAS_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef struct atlas_ctx atlas_ctx;

typedef enum {
  ATLAS_C128 = 0, /* complex128: 2 x fp64 per amplitude (P:L1964 footnote) */
  ATLAS_C64 = 1   /* complex64: 2 x fp32 per amplitude                     */
} atlas_dtype;

typedef enum {
  ATLAS_OK = 0,
  ATLAS_E_INVALID = 1,     /* bad argument: n<1, world not a power of 2,
                              G>n, qubit out of range, duplicate operand     */
  ATLAS_E_UNSUPPORTED = 2, /* unknown gate kind / option                     */
  ATLAS_E_INFEASIBLE = 3,  /* a gate has more non-insular qubits than L, or
                              no staging within s_max (P:L1526 loop)         */
  ATLAS_E_BUDGET = 4,      /* search budget exceeded                         */
  ATLAS_E_OOM = 5,         /* device/host allocation failed                  */
  ATLAS_E_CUDA = 6,        /* CUDA runtime error (or no CUDA device)         */
  ATLAS_E_NCCL = 7,        /* NCCL error / library not loadable              */
  ATLAS_E_ORDER = 8        /* call order violated (run before plan, ...)     */
} atlas_status;

/* Gate kinds.  Parameters p[] in radians. */
enum {
  ATLAS_GATE_H = 0, ATLAS_GATE_X = 1, ATLAS_GATE_Y = 2, ATLAS_GATE_Z = 3,
  ATLAS_GATE_S = 4, ATLAS_GATE_SDG = 5, ATLAS_GATE_T = 6, ATLAS_GATE_TDG = 7,
  ATLAS_GATE_RX = 8,   /* p0 = theta                                      */
  ATLAS_GATE_RY = 9,   /* p0 = theta                                      */
  ATLAS_GATE_RZ = 10,  /* p0 = theta: diag(e^{-i t/2}, e^{i t/2})          */
  ATLAS_GATE_P = 11,   /* p0 = lambda: diag(1, e^{i l})                    */
  ATLAS_GATE_U3 = 12,  /* p0..2 = theta, phi, lambda                       */
  ATLAS_GATE_CX = 13, ATLAS_GATE_CZ = 14,
  ATLAS_GATE_CP = 15,  /* p0 = lambda                                      */
  ATLAS_GATE_CCX = 16, ATLAS_GATE_SWAP = 17,
  ATLAS_GATE_CU = 18,  /* OpenQASM 3 cu(theta, phi, lambda, gamma)         */
  ATLAS_GATE_NKINDS = 19
};

/* One gate.  nq must equal the kind's arity; q[nq..2] and unused p[] are
 * ignored.  48 bytes, naturally aligned. */
typedef struct {
  uint32_t kind;
  uint32_t nq;
  uint32_t q[3];
  uint32_t pad_;
  double p[4];
} atlas_gate;

/* ---------------------------------------------------------------- core */

/* Create a context for an n-qubit state sharded over `world` ranks (a power
 * of two, 1..1024; beyond one 8-GPU box this serves planning studies such as
 * PAPER.md's staging comparison at 31 qubits); this process is
 * `rank`.  G = log2(world) global qubits,
 * L = n - G local qubits, R = 0.
 * nccl_uid: 128-byte ncclUniqueId from atlas_nccl_unique_id() on rank 0,
 * broadcast to all ranks; NULL when world == 1 or in virtual-world mode
 * (option "virtual_world": all ranks' shards live on this process's GPU,
 * the remap runs as device copies -- used to test W>1 plans on one GPU).
 * Host-only: no CUDA call is made here.  *out receives the context. */
atlas_status atlas_create(int n, atlas_dtype dtype, int world, int rank,
                          const void *nccl_uid, atlas_ctx **out);

/* Copy m gates (caller keeps ownership).  Validates kinds, arity, range and
 * distinctness.  Invalidates any existing plan. */
atlas_status atlas_load_circuit(atlas_ctx *ctx, const atlas_gate *gates, size_t m);

/* Partition: Stage with at most s_max stages and inter-node
 * cost factor c (Eq. P:L1477; c = 3 in the paper), then Kernelize
 * each stage with the cost model, then lower to device programs.
 * Deterministic: every rank computes the same plan.  Host-only. */
atlas_status atlas_plan(atlas_ctx *ctx, int s_max, double c);

/* Execute on this rank's GPU: initialise |0...0> (unless the
 * option "init" is 0, in which case the state written by atlas_set_state is
 * used), then for every stage: remap (if not the first) and launch its
 * kernels.  Blocks until the work on the context's stream is complete.
 * The first call allocates device memory (2^L amplitudes + an equal scratch
 * buffer when world > 1, times world in virtual-world mode). */
atlas_status atlas_run(atlas_ctx *ctx);

/* Copy amplitudes [first, first+count) of the final state, in LOGICAL index
 * order, into host_buf (count amplitudes of the context's dtype).  With
 * world > 1 (real NCCL ranks) each rank writes only the entries its shard
 * holds and leaves the others untouched; in virtual-world mode and world==1
 * every entry is written. */
atlas_status atlas_get_state(atlas_ctx *ctx, void *host_buf, uint64_t first,
                             uint64_t count);

/* Write amplitudes [first, first+count) (logical order) of the INITIAL state
 * of the next atlas_run (requires a plan: the stage-0 placement decides where
 * they go).  Use with option "init" = 0.  Entries not owned by this rank are
 * ignored.  The simulation works for arbitrary input states. */
atlas_status atlas_set_state(atlas_ctx *ctx, const void *host_buf, uint64_t first,
                             uint64_t count);

void atlas_destroy(atlas_ctx *ctx);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *atlas_last_error(void);

/* ------------------------------------------------------------- options */
/* Integer options (defaults in brackets):
 *   "kernelizer"     0 = Kernelize [0]: the cheapest valid of the
 *                    DP, OrderedKernelize and the front packing (DESIGN.md
 *                    R29); 1 = OrderedKernelize; 2 = greedy fusion
 *                    packing up to 5 qubits (the paper's baseline);
 *                    3 = front packing alone; 4 = the Kernelize DP alone
 *                    (pruning threshold T, no budget or fallback: E7)
 *   "front"          consider the front packing inside Kernelize [1]
 *   "dp_budget"      Kernelize DP state budget; beyond it the DP is abandoned
 *                    for the cheaper of the other candidates [250000];
 *                    states whose closed kernels already cost more than
 *                    that cheaper candidate are dropped (branch and bound);
 *                    <= 0: no budget.  Deterministic (same on every rank).
 *   "prune_T"        Kernelize pruning threshold T [500];
 *                    <= 0 means no pruning
 *   "ls_qubits"      least-significant physical qubits forced into every
 *                    shared-memory kernel (P:L1964 footnote: 3) [unset: the
 *                    cost model's value (5), see "ls_auto"]
 *   "ls_auto"        with ls_qubits unset and the built-in cost model, also
 *                    plan with one forced qubit fewer and keep the plan of
 *                    lower model cost (ties: the model's value), as long as
 *                    contiguous runs stay >= 256 B (fp64 4, fp32 5) [1]
 *   "shm_qubits"     override q_max_shared of the cost model [model]
 *   "fusion_qubits"  override q_max_fusion of the cost model [model]
 *   "kinds"          bit 0 fusion, bit 1 shared-memory [3]
 *   "insular_lift"   Kernelize insular-qubit relaxation [1]
 *   "attach"         Kernelize single-qubit attachment [1]
 *   "virtual_world"  1 = all ranks on this GPU (see atlas_create) [0]
 *   "init"           1 = atlas_run starts from |0...0> [1]
 *   "init_fuse"      1 = when the first launch is a plan-specialised
 *                    shared-memory kernel, it synthesises |0...0> in
 *                    registers instead of reading a memset shard [1]
 *   "timing"         1 = per-launch CUDA events (atlas_get_launches) [0]
 *   "shm_nbuf"       shared-memory tile buffers per CTA, 1..3 [1]
 *   "shm_split_dense" complex 2x2 blocks in shared-memory kernels are applied
 *                    as D1 R D2 (R real, D1/D2 diagonal, joined to the
 *                    phase's diagonal runs) [1]
 *   "shm_hoist_diag" diagonal ops move to the earliest diagonal run of their
 *                    register phase they commute back to [1]
 *   "shm_defer_scalar" plan-specialised kernels: unconditional real blocks
 *                    with entries of equal magnitude (H) run as adds; the
 *                    uniform scale is folded into a later block or applied
 *                    once before the kernel's last store [1]
 *   "shm_swz_phase"  plan-specialised kernels: a permuted phase store may pick
 *                    its own XOR swizzle of the tile layout (and the lanes
 *                    of each phase are re-chosen) so that stores and gathers
 *                    are bank-conflict free [1]
 *   "shm_tfac_min"   plan-specialised kernels: a diagonal slot factor whose
 *                    conditions on the thread's tile bits number at least
 *                    this many is evaluated once per thread into a shared
 *                    table (0 = never) [4]
 *   "shm_pipe"       plan-specialised kernels with one tile buffer: one CTA
 *                    per SM of two thread groups sharing a ring of three
 *                    tile buffers (loads complete on mbarriers) [1]
 *   "shm_ctas"       plan-specialised kernels of 2^12-amplitude fp64 tiles:
 *                    resident CTAs per SM, 2 (128 registers) or 3 (80
 *                    registers, when their shared memory fits) [2]
 *   "shm_const_pool" plan-specialised fp64 kernels read their gate
 *                    coefficients from a __constant__ table (LDCU.128 into
 *                    uniform registers, two per instruction) instead of
 *                    literals materialised by UMOV pairs; ptxas hoists the
 *                    loads out of the tile loop and spills at the
 *                    128-register cap, so it is off by default [0]
 *   "shm_autotune"   plan-specialised kernels: every shared-memory launch
 *                    gets up to four variants compiled (fp64 tile pipeline: two
 *                    thread groups on a ring of three buffers or two
 *                    single-buffer CTAs per SM; last phase stored straight
 *                    to HBM or through shared memory); the first atlas_run
 *                    calls after a plan time one variant each (CUDA events)
 *                    and the fastest is kept for that launch [1]
 *   "async"          1 = atlas_run, and atlas_set_state / atlas_get_state
 *                    when the layout is the identity (contiguous copies),
 *                    return once the work is enqueued on the context's
 *                    stream (atlas_set_stream) without synchronising it; the
 *                    caller synchronises that stream before it touches the
 *                    host buffers or the result (lets two contexts overlap
 *                    host<->device copies with compute) [0]
 *   "zero_lazy"      with zero_skip: when every stage-0 launch until each
 *                    local slot has been active is modelled by the tracking,
 *                    the first launch stores only tile 0 (not the zeros) and
 *                    later launches take the elements of the still-zero
 *                    region as zero in their first gather; the launch that
 *                    covers the last such slot rewrites the whole shard [1]
 *   "zero_skip"      1 = a run that starts from |0...0> tracks the local
 *                    slots no launch has made active yet (they are still 0):
 *                    an in-place plan-specialised shared-memory launch does
 *                    not visit the tiles with a 1 on such a slot (zeros in,
 *                    zeros out), and a shard that is all zero skips its
 *                    launches until the first remap [1]
 *   "shm_tma"        plan-specialised fp64 kernels of the two-group pipeline
 *                    load each tile with one TMA tensor copy
 *                    (cp.async.bulk.tensor, 128-B swizzle, mbarrier
 *                    transaction count) instead of 16 cp.async per thread,
 *                    when the launch's local slots form <= 5 runs.
 *                    Experimental: measured no faster than cp.async (qft
 *                    n = 28 2.267 vs 2.273 ms) and some n = 28 runs stall
 *                    on a tile that never completes (the kernel traps after
 *                    ~10 s), so off by default [0]
 *   "shm_fold_perm"  plan-specialised kernels: a leading register phase that
 *                    carries only a folded permutation (X/CX/SWAP) is not
 *                    run; the tile load writes every element straight to its
 *                    permuted position (one shared-memory round trip fewer)
 *                    [1]
 *   "shm_addr_split" plan-specialised kernels address a phase's shared-memory
 *                    elements as (x ^ low) + high: one pointer per distinct
 *                    low (bank-bit) part, immediate offsets for the rest [1]
 *   "shm_lit_smem"   plan-specialised fp64 kernels read the per-element
 *                    complex factors of their diagonal runs from a table in
 *                    shared memory (one broadcast LDS.128 per element instead
 *                    of four UMOVs materialising two literals); measured
 *                    slower (the kernels are shared-memory/MIO bound, not
 *                    issue bound), so off by default [0]
 *   "offload"        R > 0: host-DRAM tier (NEXT-4; the paper's regional
 *                    qubits in DRAM, Def. P:L1405-1417): the
 *                    state lives in two pinned host buffers of 2^n
 *                    amplitudes; planned as 2^R shards of 2^(n-R) whose
 *                    non-local qubits are regional; every stage streams each
 *                    shard through the GPU (H2D gathers perform the remap's
 *                    exchange, kernels, pack, D2H).  Needs world = 1; set
 *                    before the first run [0]
 *   "inplace_remap"  1 = no second shard buffer: every remap runs in place
 *                    (the pack as bit transpositions, each an in-place
 *                    pair-swap pass; the exchange as pairwise block swaps,
 *                    through a 256 MiB receive staging buffer with NCCL) --
 *                    halves the HBM a rank needs (NEXT-3: n = 36 fp64 on 8
 *                    B200s, 128 GiB shards); set before the first run [0]
 *   "shm_fuse_exchange" the remap's exchange is fused into the previous
 *                    stage's last shared-memory launch as well: it stores
 *                    each packed block straight into the buffer of the rank
 *                    it goes to -- another slot's buffer in a virtual world,
 *                    a peer GPU's memory over NVLink (CUDA IPC handles
 *                    exchanged over NCCL at the first run) with one process
 *                    per GPU, followed by a 4-byte allreduce -- so no
 *                    separate all-to-all runs.  Remaps without a pack get an
 *                    identity pack.  Needs every slot's last launch to be a
 *                    plan-specialised shared-memory kernel; library-owned
 *                    buffers for one process per GPU [1]
 *   "shm_fuse_pack"  the local bit permutation ("pack") that precedes a
 *                    remap's exchange is folded into the store addresses of
 *                    the previous stage's last shared-memory launch, which
 *                    then writes to the other buffer (no standalone pack
 *                    pass) [1]
 *   "shm_grid"       > 0: launch every shared-memory kernel on at most this
 *                    many CTAs (each then loops over many tiles; parity
 *                    tests exercise the multi-tile pipeline at small n);
 *                    0 = the occupancy-derived grid [0]
 *   "shm_jit"        1 = each shared-memory launch runs a kernel generated
 *                    from its lowered op program and compiled with NVRTC for
 *                    sm_100a at the first atlas_run after a plan (cached per
 *                    process by source); 0 = the generic interpreting
 *                    kernel.  E_CUDA if libnvrtc.so.12 cannot be loaded. [1]
 *   "shm_rb"         register bits per phase for 2^12 tiles, 3 or 4 [4]
 *   "shm_direct_store"  last phase stores straight to HBM when coalesced [1]
 *   "shm_explicit_perm" execute permutation gates in registers when a
 *                    later dense op needs their bits (else folded) [0]
 *   "device"         CUDA device ordinal [current device]
 *   "stage_budget"   staging search state budget [2000000]
 *   "regional"       R: of the log2(world) rank bits, R count as regional
 *                    qubits and the rest as global in the staging objective
 *                    (Eq. P:L1491: newly local + c * newly global; Def.
 *                    P:L1405-1417).  On one NVSwitch box the data movement
 *                    is the same all-to-all either way; R > 0 emulates a
 *                    two-tier interconnect so that c changes plans
 *                    (R7) [0]
 *   "stager"         0 = exact staging (the ILP optimum);
 *                    1 = the SnuQS greedy heuristic (the paper's staging
 *                    baseline; R32) [0]
 * String options:
 *   "cost_model"     path of a cost-model JSON (SPEC S:L358 format, integer
 *                    units); default: the built-in B200 fp64/fp32 model
 * Return ATLAS_E_UNSUPPORTED for unknown keys. */
atlas_status atlas_set_option_int(atlas_ctx *ctx, const char *key, int64_t value);
atlas_status atlas_set_option_str(atlas_ctx *ctx, const char *key, const char *value);

/* --------------------------------------------------------- plumbing */

/* Borrow device buffers owned by the caller (e.g. PyTorch tensors): `state`
 * and `scratch` each of `bytes` >= 2^L * sizeof(amplitude) (x world in
 * virtual-world mode); scratch may be NULL when world == 1. */
atlas_status atlas_bind_buffers(atlas_ctx *ctx, void *state, void *scratch,
                                uint64_t bytes);

/* Run on the given cudaStream_t (borrowed; NULL = the context's own stream). */
atlas_status atlas_set_stream(atlas_ctx *ctx, void *cuda_stream);

/* 128-byte ncclUniqueId for atlas_create (rank 0 calls it, then broadcasts).
 * Loads libnccl.so.2 at run time. */
atlas_status atlas_nccl_unique_id(void *out128);

/* ---------------------------------------------------------- reports */

/* The plan as JSON (stages with local/global logical sets, gate->stage map,
 * physical placement, per-stage kernels {gates, kind, qubits, cost}, totals).
 * Writes at most cap bytes (NUL-terminated when it fits); *len receives the
 * full length (call with cap = 0 to size). */
atlas_status atlas_get_plan_json(atlas_ctx *ctx, char *buf, size_t cap, size_t *len);

/* Plan summary, int64 values in this order (count = min(cap, 14)):
 *   0 stages  1 staging cost x1000  2 kernels  3 fusion kernels  4 shm kernels
 *   5 kernel cost total  6 remaps  7 plan time (us)  8 staging exact (1/0)
 *   9 L  10 G  11 device launches per run
 *   12 time (us) the first atlas_run after this plan spent generating,
 *      compiling (NVRTC) and loading the plan-specialised shared-memory
 *      kernels (option "shm_jit"; 0 before that run)
 *   13 staging time (us) within 7 (0 when the staging of an identical
 *      request was reused) */
atlas_status atlas_plan_stats(atlas_ctx *ctx, int64_t *out, int cap);

/* The CUDA source of the plan-specialised kernel of shared-memory launch
 * `index` (0-based, in launch order) of simulated rank `slot` (0 unless
 * virtual_world): the lowered op program of P:L1964's shared-memory kernel
 * written out as straight-line code (jit.cpp).  Host only; same buffer
 * convention as atlas_get_plan_json.  E_INVALID if there is no such launch,
 * E_ORDER before atlas_plan. */
atlas_status atlas_get_jit_source(atlas_ctx *ctx, int slot, int index, char *buf,
                                  size_t cap, size_t *len);

/* Per-launch records of the last atlas_run (needs option "timing" = 1):
 * ms[i] device time, kind[i] (0 init, 1 fused, 2 shm, 3 pack, 4 exchange,
 * 5 scale, 6 host-to-device and 7 device-to-host shard copies of the
 * offload tier), bytes[i] algorithmic HBM bytes of that launch (read + write of
 * the amplitudes it touches).  *count receives the number of records. */
atlas_status atlas_get_launches(atlas_ctx *ctx, float *ms, int32_t *kind,
                                int64_t *bytes, int cap, int *count);

/* One transfer of this rank's part of a remap exchange (the all-to-all of
 * Alg. Execute's Shard): kind 0 = send `bytes` from
 * src_off of the (packed) shard to `peer`; 1 = receive `bytes` from `peer`
 * into dst_off of the new shard; 2 = local copy src_off -> dst_off (the
 * 2^-g' share that stays on this rank).  Offsets are byte offsets into this
 * rank's shard buffers. */
typedef struct {
  int32_t peer;
  int32_t kind;
  uint64_t src_off;
  uint64_t dst_off;
  uint64_t bytes;
} atlas_xfer;

/* The exchange schedule of the remap before stage `stage` (1 <= stage < s)
 * for this context's rank -- exactly the transfers atlas_run issues (NCCL
 * grouped send/recv, or device copies in virtual-world mode).  Host-only
 * (needs a plan, no GPU).  Writes min(cap, total) records; *count = total
 * (call with cap = 0 to size).  E_INVALID for a stage out of range. */
atlas_status atlas_remap_schedule(atlas_ctx *ctx, int stage, atlas_xfer *out, int cap,
                                  int *count);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* ATLAS_H_ */
