// device.h -- POD structures shared by the host lowering and the CUDA kernels.
#pragma once
#include <cstdint>

namespace atlas {

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
enum ShmOpType : int32_t {
  OP_DIAG = 0,   // multiply by ph[sel]           (no target)
  OP_DENSE1 = 1, // 2x2 block on register bit t0, applied where sel == selv
  OP_PERM1 = 2,  // swap pair on register bit t0 (X-type), where sel == selv
  OP_DENSE2 = 3, // 4x4 block on register bits (t0 = low, t1 = high), sel == selv
};

enum SelSrc : int32_t { SEL_REG = 0, SEL_THR = 1, SEL_BASE = 2 };

struct ShmOp {
  int32_t type;
  int32_t t0, t1;          // register-bit indices of the targets
  int32_t nsel;            // number of selector bits (<= 3)
  int32_t sel_src[3];      // SelSrc
  int32_t sel_idx[3];      // REG: register bit; THR: tile bit; BASE: physical slot
  int32_t selv;            // DENSE/PERM: selector value on which the block acts
  int32_t pad;
  double m[32];            // DIAG: ph[2^nsel] (re,im); DENSE1: 2x2; DENSE2: 4x4
};

struct ShmPhase {
  int32_t rbit[4];         // tile bits held in registers (RB used)
  int32_t op_begin, op_end;
};

struct ShmLaunch {
  int32_t K, RB;           // tile bits, register bits
  int32_t c0;              // leading contiguous active slots (act[i] == i for i < c0)
  int32_t nphase;
  uint64_t nonactive;      // mask of non-active local slots (tile base bits)
  uint64_t ntiles;
  int64_t hightab_off;     // offset (elements of uint64) into the table blob
  int64_t ops_off;         // offset (ShmOp) into the op blob
  int64_t phase_off;       // offset (ShmPhase) into the phase blob
};

// Fused dense kernel ("Fusion"): one 2^k x 2^k matrix on k slots.
struct FusedLaunch {
  int32_t k;
  int32_t t[6];            // physical target slots, ascending; matrix bit j <-> t[j]
  int32_t pad;
  int64_t mat_off;         // offset (complex elements) into the matrix blob
};

}  // namespace atlas
