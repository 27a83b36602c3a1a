// ctx.h -- the atlas_ctx object: circuit, plan, lowered device programs.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "device.h"
#include "internal.h"

namespace atlas {

enum LaunchType { L_INIT = 0, L_FUSED = 1, L_SHM = 2, L_PACK = 3, L_EXCHANGE = 4, L_SCALE = 5,
                  L_H2D = 6, L_D2H = 7 };

struct Launch {
  int type = 0;
  int stage = 0;
  FusedLaunch fl{};
  ShmLaunch sl{};
  int64_t newpos_off = -1;   // L_PACK: offset into newpos blob (L ints)
  double sre = 1, sim = 0;   // L_SCALE
  int64_t bytes = 0;         // algorithmic HBM bytes
  void *jit = nullptr;       // L_SHM: plan-specialised kernel (jit.cpp), or null
  // autotuning (option shm_autotune): the variants of the same launch (tile
  // pipeline x direct last-phase store; variant 0 = the defaults) and the
  // device time each took in the tuning runs; nvar = 0 once tuned
  void *jit_var[4] = {nullptr, nullptr, nullptr, nullptr};
  float tune_ms[4] = {-1.f, -1.f, -1.f, -1.f};
  int nvar = 0;
  bool tune_warm = false;  // the first run after the JIT runs variant 0 untimed (cold pages, first launches)
};

// Exchange of one remap (stage boundary k-1 -> k): swap the g' top local
// slots with the incoming qubits' global slots.
struct Exchange {
  int gp = 0;                   // g'
  std::vector<int> gamma;       // global slot offsets (slot - L) of incoming qubits, j-th
  std::vector<int> fI;          // flip of the j-th incoming qubit before the exchange
  bool packed = false;          // a pack launch precedes (source = scratch)
};

// one transfer of a rank's part of a remap exchange
enum XferKind { XFER_SEND = 0, XFER_RECV = 1, XFER_LOCAL = 2 };
struct Xfer {
  int peer;            // the other rank (this rank for XFER_LOCAL)
  int kind;
  uint64_t src_off;    // byte offset in the (packed) source shard (send, local)
  uint64_t dst_off;    // byte offset in the destination shard (recv, local)
  uint64_t bytes;
};

struct StageMap {
  std::vector<int> sigma;       // logical -> physical slot during the stage
  std::vector<int> flip_end;    // per logical qubit: flip bit at the end of the stage
  std::vector<int> flip_begin;  // at the start
};

struct Options {
  int kernelizer = 0;
  int prune_T = 500;
  int ls_qubits = 5;
  int ls_auto = 1;           // ls_qubits unset: also try one fewer, keep the cheaper plan
  int shm_qubits = -1;
  int fusion_qubits = -1;
  int kinds = 3;
  int lift = 1;
  int attach = 1;
  int virtual_world = 0;
  int init = 1;
  int init_fuse = 1;         // |0...0> synthesised by the first SHM kernel (no memset pass)
  int timing = 0;
  int device = -1;
  long stage_budget = 2000000;
  int regional = 0;          // rank bits counted as regional qubits in the staging cost (R > 0 emulation)
  int stager = 0;            // 0: exact staging (ILP optimum); 1: SnuQS greedy baseline (E5)
  int shm_nbuf = 1;
  int shm_direct_store = 1;
  int shm_rb = 4;
  int shm_explicit_perm = 0;
  int front = 1;
  int shm_split_dense = 1;   // complex 2x2 blocks -> D1 R D2 (real R) in SHM kernels
  int shm_hoist_diag = 1;    // diagonal ops join the earliest reachable diagonal run
  int shm_hoist_dense = 1;   // dense ops join the earliest dense item they commute back to
  int shm_defer_diag = 1;    // diagonal ops on non-register bits wait for the next phase if one starts
  int shm_defer_scalar = 1;  // JIT: H-type blocks as adds, their uniform scale deferred
  int shm_swz_phase = 1;     // JIT: per-boundary SMEM swizzles for permuted stores
  int shm_tfac_min = 4;      // JIT: thread-only factor tables for slots with >= this many entries (0: off)
  int shm_pipe = 1;          // JIT: two thread groups per CTA on a ring of 3 tile buffers
  int shm_ctas = 2;          // JIT: resident SHM CTAs per SM for 2^12 fp64 tiles (2 or 3)
  int inplace_remap = 0;     // remaps in place (pair swaps), no scratch shard buffer (NEXT-3)
  int shm_fuse_exchange = 1; // the fused-pack launch also stores each block into its destination rank's buffer
  int shm_fuse_pack = 1;     // the remap pack fused into the previous stage's last SHM launch
  int shm_grid = 0;          // > 0: cap every SHM launch at this many CTAs (tests: many tiles per CTA at small n)
  int shm_const_pool = 0;    // JIT fp64: coefficients in a __constant__ table (c[] operands, no UMOV)
  int shm_tma = 0;           // JIT fp64 pipe: tile loads as one TMA tensor copy (experimental, off: see DESIGN 5e)
  int shm_fold_perm = 1;     // JIT: a leading permutation-only phase folded into the tile load
  int shm_addr_split = 1;    // JIT: shared-memory addresses as (x ^ low) + high (immediate offsets)
  int shm_lit_smem = 0;      // JIT fp64: diagonal-run element factors read from a shared-memory table
  int shm_autotune = 1;      // JIT fp64: time both tile pipelines per launch in the first runs, keep the faster
  int async = 0;             // run / set_state / get_state (contiguous layouts) return without a stream sync
  int zero_lazy = 1;         // with zero_skip: zeros of the |0...0> launch not stored, zero-filled on load
  int zero_skip = 1;         // runs from |0...0>: tiles provably zero in and out are not visited
  int shm_jit = 1;           // 1: plan-specialised SHM kernels (NVRTC); 0: interpreter
  long long dp_budget = 250000;
  std::string cost_model;
};

struct NcclApi;

}  // namespace atlas

struct atlas_ctx {
  int n = 0, world = 1, rank = 0, G = 0, L = 0;
  atlas_dtype dt = ATLAS_C128;
  atlas::Options opt;
  unsigned char nccl_uid[128];
  bool have_uid = false;

  std::vector<atlas::Gate> gates;
  std::vector<atlas::GateInfo> info;

  // plan
  bool planned = false;
  double plan_us = 0;
  double stage_us = 0;         // staging part of plan_us
  double c = 3;
  atlas::CostModel cm;
  atlas::StagePlan sp;
  // key of the staging in sp (invalidated by atlas_load_circuit)
  bool sp_key_valid = false;
  int sp_key_smax = 0;
  double sp_key_c = 0;
  long sp_key_budget = 0;
  int sp_key_stager = 0;
  int sp_key_regional = 0;
  std::vector<atlas::StageMap> maps;
  std::vector<std::vector<int>> stage_gates;     // circuit ids per stage (order)
  std::vector<atlas::KernelPlan> kplans;         // per stage; gate ids = circuit ids
  std::vector<atlas::Exchange> exch;             // per stage (index 0 unused)
  int K_tile = 0;

  // lowered programs: one per simulated rank (world in virtual mode, else 1)
  int nslots = 1;
  std::vector<std::vector<atlas::Launch>> prog;
  std::vector<double> coef;
  std::vector<atlas::ShmOp> ops;
  std::vector<atlas::ShmPhase> phases;
  std::vector<atlas::DiagEnt> ents;
  std::vector<atlas::PermTerm> terms;
  std::vector<double2> mats;
  std::vector<int> newpos;

  // device
  bool dev_ready = false, blobs_ready = false, jit_ready = false;
  double jit_us = 0;          // generation + NVRTC compile + load of the SHM kernels
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<void *> d_state, d_scratch;  // per slot (no scratch with option inplace_remap)
  void *d_stage = nullptr;                 // in-place remap receive staging (multi-process)
  // host-DRAM offload tier (option offload = R, NEXT-4): the 2^R shards
  // ("regional" chunks, Def. P:L1405-1417) live in two pinned host buffers
  // (ping-pong across stages); each stage streams every shard through the
  // two device work buffers
  int offload = 0;
  void *h_buf[2] = {nullptr, nullptr};
  int h_cur = 0;
  void *d_work[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  std::vector<int> cur;                    // 0: state holds the data, 1: scratch
  bool bound = false;
  void *d_coef = nullptr, *d_ops = nullptr, *d_phases = nullptr, *d_mats = nullptr,
       *d_newpos = nullptr, *d_ents = nullptr, *d_terms = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<float> launch_ms;
  std::vector<int> launch_kind;
  std::vector<int64_t> launch_bytes;
  void *nccl_comm = nullptr;
  // fused exchange over peer memory (option shm_fuse_exchange, one process
  // per GPU): every rank's state and scratch shard opened by CUDA IPC
  bool ipc_ready = false;
  std::vector<void *> ipc_state, ipc_scratch;  // [rank]; own rank = own buffers
  void *d_bar = nullptr;                       // 4 B: the allreduce that ends a fused exchange
  bool state_set = false;
};
