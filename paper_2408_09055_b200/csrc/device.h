// device.h -- POD structures shared by the host lowering and the CUDA kernels.
#pragma once
#include <cstdint>

namespace atlas {

#ifdef __CUDACC__
#define ATLAS_HD __host__ __device__
#else
#define ATLAS_HD
#endif

// XOR swizzle of a shared-memory tile index so that the 8 (fp64) / 16 (fp32)
// lanes of one shared-memory wavefront hit distinct 16-byte bank groups for
// the access patterns of the load/store loops and of most register phases.
// It is linear over GF(2): swz(a ^ b) = swz(a) ^ swz(b).
ATLAS_HD constexpr int swz_c128(int j) { return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9) ^ (j >> 12)) & 7); }
ATLAS_HD constexpr int swz_c64(int j) { return j ^ (((j >> 4) ^ (j >> 8) ^ (j >> 12)) & 15); }

// ----------------------------------------------------------------------------
// Shared-memory kernel program ("Shared-memory": load a
// micro-batch into shared memory and apply the gates one by one).
//
// A tile is 2^K amplitudes whose index bits are the K *active* physical
// qubits; tile bit b <-> physical slot act[b].  The ops of the
// kernel are grouped into register phases: in phase p every thread holds
// 2^RB amplitudes in registers whose tile bits are phase.rbit[0..RB-1]; an op
// may only target register bits.  Selector bits (controls and diagonal
// qubits, i.e. the gate's insular operands) may be any local qubit: a
// register bit, a thread bit of the tile, or a non-active qubit whose value
// is known per tile ("converts these gates into smaller gates with
// only active qubits").
// ----------------------------------------------------------------------------
enum ShmOpType : uint8_t {
  OP_PHASE = 0,   // v[e] *= c on masked elements   (generic diagonal fallback)
  OP_DENSE1 = 1,  // 2x2 block on register bit t0
  OP_PERM1 = 2,   // swap on register bit t0 (X-type block; non-affine fallback)
  OP_DENSE2 = 3,  // 4x4 block on register bits t0 < t1
  OP_DIAG = 4,    // diagonal accumulator of one factor slot (see below)
};

// Op flags
enum : uint8_t {
  OPF_FULL = 1,   // unconditional: every register element, every thread, every tile
  OPF_REAL = 2,   // OP_DENSE1 whose 2x2 block is real (H, RY, ...): half the flops
};

// One op of a shared-memory kernel.  It acts on the register elements e with
// bit e of emask set, in threads whose fixed tile bits
// satisfy (jt & thr_mask) == thr_val, in tiles whose base satisfies
// (base & base_mask) == base_val -- i.e. the selector (control / diagonal)
// values of the gate.
//
// OP_DIAG (a run of diagonal gates, DESIGN.md §5 "diagonal accumulator"):
// t0 = factor slot s: 0 = F (every element), 1..RB = K_i (elements with
// register bit i-1 set), 5.. = P_ij (elements with register bits i and j set,
// pairs in the order (0,1),(0,2),(0,3),(1,2),(1,3),(2,3)).  The factor is
// coef[coef] (the product of the run's unconditional contributions) times
// the c of every DiagEnt in [base_mask, base_val) whose thread/tile condition
// holds.  A diagonal gate whose register selectors number <= 2 decomposes
// exactly into such factors (x_a x_b products of selector indicators).
struct ShmOp {
  uint8_t type, t0, t1, flags;
  uint16_t emask;              // register-bit condition as a mask over e (or pair/quad base e)
  uint16_t pad2;
  uint16_t thr_mask, thr_val;
  int32_t coef;                // offset (doubles) into the launch's coefficients
  uint64_t base_mask, base_val;  // OP_DIAG: entry range [base_mask, base_val)
};
static_assert(sizeof(ShmOp) == 32, "ShmOp layout");

// conditional factor of an OP_DIAG slot
struct DiagEnt {
  uint16_t thr_mask, thr_val;
  uint32_t has_base;
  uint64_t base_mask, base_val;
  double re, im;
};
static_assert(sizeof(DiagEnt) == 40, "DiagEnt layout");

// Affine permutation gates (X, CX, SWAP and base-controlled CX) of a phase
// are not executed: they are folded into the phase's store addresses.  The
// value held for tile index j is stored at tile index A j ^ c(base), with
// c(base) = c0 ^ XOR of the PermTerm vectors whose base condition holds.
// colimg[b] = swz(A e_b) (the swizzle is linear, so addresses are XORs).
struct PermTerm {
  uint64_t base_mask, base_val;
  uint64_t gvec;               // the vector deposited on the physical slots
  uint32_t vec_swz, pad;       // swizzled tile vector
};
static_assert(sizeof(PermTerm) == 32, "PermTerm layout");

struct ShmPhase {
  int32_t rbit[4];             // tile bits held in registers (RB used)
  int32_t op_begin, op_end;
  uint16_t colimg[16];         // store image of each tile bit (swizzled)
  uint32_t c0_swz;             // swizzled constant of the store map
  int16_t permuted;            // 0: identity store (colimg/c0 unused)
  // tile bits of thread bits 0..W-1 (W = 3 fp64 / 4 fp32: the lanes of one
  // shared-memory wavefront), one nibble each, 0xF = unused; 0xFFFF = the
  // default (non-register tile bits in ascending order).  Chosen so that the
  // gather and the permuted store of the phase are bank-conflict free.
  uint16_t qlane;
  int32_t term_begin, term_end;
};
static_assert(sizeof(ShmPhase) == 72, "ShmPhase layout");

struct ShmLaunch {
  int32_t K, RB, nphase, nops, ncoef, nbuf;  // nbuf: 1 or 2 tile buffers
  int32_t act[16];             // tile bit b <-> physical slot act[b] (ascending)
  uint64_t nonactive;          // mask of the non-active local slots
  uint64_t ntiles;
  int64_t ops_off, coef_off, phase_off;
  int64_t ent_off, term_off;
  int32_t nent, nterm;
  // last_direct: the last phase stores its registers straight to HBM (no
  // shared-memory round trip); chosen when its register bits avoid the 5
  // lowest tile bits, so the lanes of a warp cover contiguous 512-B runs.
  // lcol[b] = physical offset of tile bit b under the last phase's folded
  // map (1 << act[b] when it is the identity), lc0 = offset of its constant.
  int32_t last_direct;
  int32_t grid_cap;            // > 0: at most this many CTAs (option shm_grid; tests)
  uint64_t lcol[16];
  uint64_t lc0;
  // >= 0: the fused remap pack (plan.cpp, option shm_fuse_pack): offset of
  // the L-entry slot map in the newpos blob; the launch then writes to the
  // other buffer with local slot b moved to newpos[b] (plan-specialised
  // kernels only; the interpreter runs in place and a permute follows)
  int64_t out_perm_off;
  // > 0 (with out_perm_off): the launch also performs the next remap's
  // exchange (option shm_fuse_exchange): output offset y goes to
  // peers[y >> (L - peer_gp)][y & (2^(L - peer_gp) - 1)], the 2^peer_gp
  // destination blocks (the peers' other buffers, or this slot's own) passed
  // as a launch argument
  int32_t peer_gp;
  // 1: the launch may run with lazy zeros (zfill != 0: it lies in stage 0
  // between the |0...0> launch and the launch that makes every local slot
  // active); only such kernels carry the zero-fill load code
  int32_t zfill_cap;
};

// Fused dense kernel ("Fusion"): one 2^k x 2^k matrix on k slots.
struct FusedLaunch {
  int32_t k;
  int32_t t[6];            // physical target slots, ascending; matrix bit j <-> t[j]
  int32_t pad;
  int64_t mat_off;         // offset (complex elements) into the matrix blob
};

}  // namespace atlas
