// kernelize.cpp -- OrderedKernelize and the greedy baseline.
//
// Cost model (PAPER.md §"Cost Function in Kernelize"):
//   fusion kernel        fusion_cost[|Qubits(K)|]
//   shared-memory kernel alpha + sum_{g in K} Cost(g)
// Qubits are the stage-local qubits of the gates (R13).  A
// shared-memory kernel's active set is the union of its gates' non-insular
// local qubits plus the ls forced least-significant physical
// qubits (P:L1964 footnote); it must fit q_max_shared.  Kinds are tried in
// the order fusion, shared memory; a tie keeps fusion.
#include <algorithm>
#include <climits>

#include "internal.h"

namespace atlas {

static const int64_t INF64 = LLONG_MAX / 4;

struct Caps {
  int qmf, qms;
};
static Caps caps(const CostModel &cm, const KernelizeOptions &o) {
  Caps c;
  c.qmf = (o.kinds & 1) ? std::min(cm.q_max_fusion, o.L) : 0;
  c.qms = (o.kinds & 2) ? std::min(cm.q_max_shared, o.L) : -1;
  if (c.qms >= 0 && c.qms < 6) c.qms = -1;  // device tiles need >= 6 active qubits
  return c;
}

static int64_t cost_of(u64 qubits, u64 active, int64_t gsum, const CostModel &cm, Caps c,
                       int *kind) {
  const int q = popc(qubits);
  int64_t f = (q >= 1 && q <= c.qmf) ? cm.fusion_cost[q - 1] : INF64;
  int64_t s = (popc(active) <= c.qms) ? cm.alpha + gsum : INF64;
  if (f <= s) {
    if (kind) *kind = K_FUSION;
    return f;
  }
  if (kind) *kind = K_SHM;
  return s;
}

int64_t kernel_cost(const std::vector<KGate> &seq, const std::vector<int> &idx,
                    const CostModel &cm, const KernelizeOptions &o, int *kind) {
  u64 q = 0, a = o.ls_set;
  int64_t gs = 0;
  for (int i : idx) {
    q |= seq[i].qubits;
    a |= seq[i].active;
    gs += cm.gate_cost[seq[i].kind];
  }
  return cost_of(q, a, gs, cm, caps(cm, o), kind);
}

static Kernel make_kernel(const std::vector<KGate> &seq, int a, int b, int kind,
                          const KernelizeOptions &o, int64_t cost) {
  Kernel K;
  K.kind = kind;
  K.cost = cost;
  u64 q = 0, act = o.ls_set;
  for (int i = a; i < b; i++) {
    K.gates.push_back(i);
    q |= seq[i].qubits;
    act |= seq[i].active;
  }
  K.qubits = kind == K_FUSION ? q : act;
  return K;
}

// Alg. OrderedKernelize: DP[i+1] = min_j DP[j] + Cost(C[j..i]).
// Ties keep the smallest j (R21).
KernelPlan ordered_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                             const KernelizeOptions &o) {
  const int m = (int)seq.size();
  const Caps c = caps(cm, o);
  std::vector<int64_t> dp(m + 1, INF64);
  std::vector<int> from(m + 1, -1), kindv(m + 1, 0);
  dp[0] = 0;
  for (int i = 0; i < m; i++) {
    u64 q = 0, a = o.ls_set;
    int64_t gs = 0;
    for (int j = i; j >= 0; j--) {
      q |= seq[j].qubits;
      a |= seq[j].active;
      gs += cm.gate_cost[seq[j].kind];
      const bool fus_ok = popc(q) <= c.qmf;
      const bool shm_ok = popc(a) <= c.qms;
      if (!fus_ok && !shm_ok) break;  // supersets stay infeasible
      if (dp[j] >= INF64) continue;
      int kind;
      int64_t cst = cost_of(q, a, gs, cm, c, &kind);
      if (cst >= INF64) continue;
      if (dp[j] + cst <= dp[i + 1]) {
        dp[i + 1] = dp[j] + cst;
        from[i + 1] = j;
        kindv[i + 1] = kind;
      }
    }
    if (dp[i + 1] >= INF64) fail(ATLAS_E_INFEASIBLE, "gate %d fits no kernel kind", seq[i].gid);
  }
  KernelPlan kp;
  kp.total = dp[m];
  std::vector<Kernel> rev;
  for (int e = m; e > 0; e = from[e]) {
    int b = from[e];
    rev.push_back(make_kernel(seq, b, e, kindv[e], o, dp[e] - dp[b]));
  }
  kp.kernels.assign(rev.rbegin(), rev.rend());
  return kp;
}

// The paper's kernelization baseline: pack gates left to right into
// fusion kernels of up to 5 qubits.
KernelPlan greedy_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                            const KernelizeOptions &o) {
  const int m = (int)seq.size();
  const int cap = std::min(5, std::min(cm.q_max_fusion, o.L));
  KernelPlan kp;
  int a = 0;
  u64 q = 0;
  auto close = [&](int b) {
    if (b <= a) return;
    int64_t cst = cm.fusion_cost[std::max(1, popc(q)) - 1];
    kp.kernels.push_back(make_kernel(seq, a, b, K_FUSION, o, cst));
    kp.total += cst;
  };
  for (int i = 0; i < m; i++) {
    if (popc(q | seq[i].qubits) > cap) {
      close(i);
      a = i;
      q = 0;
    }
    q |= seq[i].qubits;
  }
  close(m);
  return kp;
}

}  // namespace atlas

namespace atlas {

// Commutation-aware greedy packing ("front" kernelizer).  Gates a < b must
// keep their order iff they share a qubit that is non-diagonal in either
// (the exact relation Thm. dp-correct's topological equivalence is checked
// with).  Kernels are built one at a time from the ready front of
// that dependency DAG: a ready gate joins the open kernel while the kernel
// still fits (shared-memory: active set incl. the forced LSB qubits <=
// q_max_shared; fusion-only: qubits <= q_max_fusion), the gate adding the
// fewest new qubits first (ties: circuit order); gates made ready by it may
// join the same kernel.  This finds column-wise packings of entangling
// blocks (e.g. su2random's all-to-all CX blocks: one kernel per window of
// target qubits across all rows) that the DP's deferred-merging heuristics
// miss; Kernelize returns the cheapest valid candidate (R29).
KernelPlan front_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                           const KernelizeOptions &o) {
  const int m = (int)seq.size();
  const Caps c = caps(cm, o);
  const bool shm = c.qms >= 0;
  const int cap = shm ? c.qms : c.qmf;
  KernelPlan kp;
  if (m == 0) return kp;
  std::vector<std::vector<int>> succ(m);
  std::vector<int> indeg(m, 0);
  for (int a = 0; a < m; a++)
    for (int b = a + 1; b < m; b++) {
      const u64 sh = seq[a].qubits & seq[b].qubits;
      if (sh && (sh & (seq[a].active | seq[b].active))) {
        succ[a].push_back(b);
        indeg[b]++;
      }
    }
  std::vector<int> ready;
  for (int g = 0; g < m; g++)
    if (!indeg[g]) ready.push_back(g);
  int done = 0;
  while (done < m) {
    Kernel K;
    u64 q = 0, act = o.ls_set;
    int64_t gs = 0;
    for (;;) {
      int best = -1, best_grow = 1 << 30, best_pos = -1;
      for (int r = 0; r < (int)ready.size(); r++) {
        const int g = ready[r];
        const u64 nq = q | seq[g].qubits, na = act | seq[g].active;
        const int size = shm ? popc(na) : popc(nq);
        if (size > cap) continue;
        const int grow = size - (shm ? popc(act) : popc(q));
        if (grow < best_grow || (grow == best_grow && g < best)) {
          best = g;
          best_grow = grow;
          best_pos = r;
        }
      }
      if (best < 0) {
        if (!K.gates.empty()) break;
        // nothing fits an empty kernel of this kind: take the earliest ready gate alone
        best_pos = 0;
        for (int r = 1; r < (int)ready.size(); r++)
          if (ready[r] < ready[best_pos]) best_pos = r;
        best = ready[best_pos];
      }
      ready.erase(ready.begin() + best_pos);
      K.gates.push_back(best);
      q |= seq[best].qubits;
      act |= seq[best].active;
      gs += cm.gate_cost[seq[best].kind];
      done++;
      for (int s2 : succ[best])
        if (--indeg[s2] == 0) ready.push_back(s2);
    }
    int kind = 0;
    K.cost = cost_of(q, act, gs, cm, c, &kind);
    K.kind = kind;
    K.qubits = kind == K_FUSION ? q : act;
    kp.total += K.cost;
    kp.kernels.push_back(K);
  }
  return kp;
}

}  // namespace atlas
