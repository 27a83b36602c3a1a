// internal.h -- shared declarations of the Atlas B200 library (host side).
#pragma once

#include <complex>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/atlas.h"

namespace atlas {

using cd = std::complex<double>;
using u64 = uint64_t;
using u32 = uint32_t;

// ---------------------------------------------------------------- errors
struct Error {
  atlas_status st;
  std::string msg;
};
[[noreturn]] void fail(atlas_status st, const char *fmt, ...);
void set_last_error(const std::string &m);

inline int popc(u64 x) { return __builtin_popcountll(x); }
inline int ctz(u64 x) { return __builtin_ctzll(x); }

// ----------------------------------------------------------------- gates
// Operand roles after insular classification (Def. Insular Qubit,
// PAPER.md P:L1430-1441):
//   TGT  non-insular (must be local; must be active in a shared-memory kernel)
//   CTL  control of a controlled-U (block-diagonal w.r.t. the qubit and the
//        identity on its |0> block); the footnote's symmetric gates (CZ, CP)
//        have every operand CTL
//   DIAG the qubit of a diagonal single-qubit gate
//   ANTI the qubit of an anti-diagonal single-qubit gate
enum Role : uint8_t { TGT = 0, CTL = 1, DIAG = 2, ANTI = 3 };

struct Gate {
  int kind;
  int nq;
  int q[3];
  double p[4];
};

struct GateInfo {
  u64 qmask = 0;      // all operands
  u64 nonins = 0;     // non-insular operands
  u64 diagtype = 0;   // operands on which the gate is block diagonal (CTL/DIAG)
  u64 antitype = 0;   // ANTI operands
  Role role[3] = {TGT, TGT, TGT};
};

int kind_arity(int kind);
const char *kind_name(int kind);
// Row-major 2^k x 2^k unitary; operand j <-> bit j of the row/column index.
void gate_matrix(const Gate &g, cd *U);
GateInfo classify(const Gate &g);

// ------------------------------------------------------------ cost model
// SPEC S:L245-253 / PAPER.md P:L1958-1968, integer units (R11).
struct CostModel {
  std::vector<int64_t> fusion_cost;  // index q-1
  int64_t alpha = 0;
  int64_t gate_cost[ATLAS_GATE_NKINDS] = {0};
  int q_max_fusion = 0;
  int q_max_shared = 0;
  int ls_qubits = 0;
  std::string source;
};
CostModel load_cost_model(const std::string &path_or_json, bool is_json);
CostModel builtin_cost_model(atlas_dtype dt);

// ------------------------------------------------------------------ plan
struct StagePlan {
  int s = 0;
  double cost = 0;
  bool exact = true;
  std::vector<u64> local;        // logical local set per stage
  std::vector<u64> global;       // logical global set per stage
  std::vector<int> gate_stage;   // per gate
  long states_explored = 0;
};

// One gate as the kernelizer sees it (R13):
struct KGate {
  int gid;          // index in the circuit
  u64 qubits;       // logical qubits local in the stage
  u64 active;       // non-insular local qubits (shared-memory active set)
  u64 diagq;        // local qubits on which the gate is diagonal-type
  u64 antiq;        // local qubits on which the gate is anti-diagonal-type
  int kind;         // original kind (cost table key)
};

enum KernelKind { K_FUSION = 0, K_SHM = 1 };

struct Kernel {
  std::vector<int> gates;  // circuit gate ids in execution order
  int kind = K_FUSION;
  u64 qubits = 0;          // logical qubits (fusion: all; shm: active + LSB)
  int64_t cost = 0;
  int nphase = 0;          // shm: register phases of the lowered program (rank 0)
};

struct KernelPlan {
  std::vector<Kernel> kernels;
  int64_t total = 0;
};

struct KernelizeOptions {
  int algo = 0;            // 0 Kernelize, 1 Ordered, 2 greedy-5, 3 front, 4 the DP alone
  int prune_T = 500;
  bool lift = true;
  bool attach = true;
  int kinds = 3;
  bool front = true;       // also consider the front packing (R29)
  long long dp_budget = 0; // Kernelize DP state budget (0 = none)
  int L = 0;               // local qubits (caps kernel sizes)
  u64 ls_set = 0;          // logical qubits at the forced LSB physical slots
};

StagePlan stage_circuit(int n, int L, int G, const std::vector<GateInfo> &info,
                        int s_max, double c, long budget, int R = 0);
StagePlan stage_greedy(int n, int L, int G, const std::vector<GateInfo> &info, int s_max, double c);

KernelPlan ordered_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                             const KernelizeOptions &o);
KernelPlan greedy_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                            const KernelizeOptions &o);
KernelPlan front_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                           const KernelizeOptions &o);
KernelPlan dp_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                        const KernelizeOptions &o);
// the DP of Alg. Kernelize alone (pruning at T, no budget, no bound, no
// fallback candidates): the planner-time / cost trade-off of E7
KernelPlan dp_only_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                             const KernelizeOptions &o);
// cost of a kernel made of these gates, best kind (fusion preferred on a tie)
int64_t kernel_cost(const std::vector<KGate> &seq, const std::vector<int> &idx,
                    const CostModel &cm, const KernelizeOptions &o, int *kind);

}  // namespace atlas
