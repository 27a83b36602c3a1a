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
enum ShmOpType : uint8_t {
  OP_PHASE = 0,   // v[e] *= c                      (diagonal gates, scalars)
  OP_DENSE1 = 1,  // 2x2 block on register bit t0
  OP_PERM1 = 2,   // swap on register bit t0 (X-type block)
  OP_DENSE2 = 3,  // 4x4 block on register bits t0 < t1
};

// One op of a shared-memory kernel.  It acts on the register elements e with
// bit e of emask set, in threads whose fixed tile bits
// satisfy (jt & thr_mask) == thr_val, in tiles whose base satisfies
// (base & base_mask) == base_val -- i.e. the selector (control / diagonal)
// values of the gate.
struct ShmOp {
  uint8_t type, t0, t1, pad;
  uint16_t emask;              // register-bit condition as a mask over e (or pair/quad base e)
  uint16_t pad2;
  uint16_t thr_mask, thr_val;
  int32_t coef;                // offset (doubles) into the launch's coefficients
  uint64_t base_mask, base_val;
};
static_assert(sizeof(ShmOp) == 32, "ShmOp layout");

struct ShmPhase {
  int32_t rbit[4];             // tile bits held in registers (RB used)
  int32_t op_begin, op_end;
};

struct ShmLaunch {
  int32_t K, RB, nphase, nops, ncoef, nbuf;  // nbuf: 1 or 2 tile buffers
  int32_t act[16];             // tile bit b <-> physical slot act[b] (ascending)
  uint64_t nonactive;          // mask of the non-active local slots
  uint64_t ntiles;
  int64_t ops_off, coef_off, phase_off;
};

// Fused dense kernel ("Fusion"): one 2^k x 2^k matrix on k slots.
struct FusedLaunch {
  int32_t k;
  int32_t t[6];            // physical target slots, ascending; matrix bit j <-> t[j]
  int32_t pad;
  int64_t mat_off;         // offset (complex elements) into the matrix blob
};

}  // namespace atlas
