// kernelize_dp.cpp -- Alg. Kernelize with the
// extensible-qubit state compression of Alg. ExtQ and the
// implementation optimisations of App. "Optimizations to the Kernelize
// Algorithm".
//
// DP state: the cost of the kernels already closed, and the ORDERED
// set KS of open kernels, each described by
//   kind (fusion / shared memory; fixed at creation),
//   Qubits(K), ExtQ(K) (ALL or a subset of Qubits(K)),
//   for shared-memory kernels the active set (non-insular qubits) and
//   the extensible-insular set, and the summed gate cost.
// Transitions for gate C[i] (here: an attachment *unit*, see below):
//   add to an open kernel K if Qubits(C[i]) are extensible for K (Constraint 1
//     via Def. 5); K keeps its place if monotonicity applies to it
//     (ExtQ != ALL), else it moves to the end;
//   or open a new singleton kernel at the end, one copy per kind.
// Then ExtQ of the other kernels is updated by Alg. ExtQ.
// Optimisations, with the readings of DESIGN.md:
//   * insular lifting: for shared-memory kernels the intersect
//     test of P:L1831 ignores qubits insular to C[i] and to every gate of K',
//     and a gate may join if its non-insular qubits are in ExtQ and its insular
//     qubits in the extensible-insular set (R16: insular = diagonal-type);
//   * subsumption: if Qubits(C[i]) and Qubits(K) are nested and
//     C[i] may join K, it joins K without branching;
//   * deferred merging: C[i] is not tried in kernels whose ExtQ
//     is ALL; when such a kernel K' loses ALL because of C[i], it may be merged
//     with one other ALL kernel of the same kind (or stay alone);
//   * attachment: single-qubit gates ride with the adjacent
//     multi-qubit gate on their qubit (successor first, else predecessor);
//     a non-diagonal attached gate makes that qubit non-insular in the unit;
//   * post-processing: the open kernels are packed greedily in
//     order: fusion kernels while the merged cost is not larger, shared-memory
//     kernels while the active set fits;
//   * pruning: when a position holds >= T states, keep the T/2
//     cheapest by (closed cost + post-processed open cost).
// Closing (line 1726's min over KS'): kernels that can no longer grow
// (ExtQ and extensible-insular sets empty) are closed as soon as they form a
// prefix of KS; a kernel that can still grow is only closed at the end
// (reading R17: closing it earlier never lowers the reachable cost).
// The realised order is checked for topological equivalence (Thm. dp-correct,
// P:L1743) under the exact commutation relation; the cheaper of this result
// and OrderedKernelize is returned (Thm. dp-optimal, guarantees the
// DP is not worse without pruning).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iterator>
#include <unordered_map>

#include "internal.h"

namespace atlas {

namespace {

const int64_t INF64 = LLONG_MAX / 4;
// deferred merging: at most this many non-host ALL partners are tried for a
// kernel that loses ALL (the most recently ordered ones; reading R18)
static int kMaxPartners = 4;
// at most this many merges along one branch for one gate; a separate greedy
// branch merges every touched ALL kernel into the host
static int kMaxMergesPerGate = 2;

struct Unit {
  u64 qubits = 0, active = 0;
  int64_t gcost = 0;
  std::vector<int> gates;  // indices into seq, execution order
};

struct KD {
  uint8_t kind = 0;
  bool all = true;
  u64 qubits = 0, extq = 0, extins = 0, active = 0;
  int64_t gcost = 0;
  int glist = -1;  // arena list of unit indices (reverse order)
  int nunits = 0;
  bool operator==(const KD &o) const {
    return kind == o.kind && all == o.all && qubits == o.qubits && extq == o.extq &&
           extins == o.extins && active == o.active && gcost == o.gcost;
  }
};

// rope of unit indices: leaf (a = unit, b = -2) or concatenation (a, b)
struct Node {
  int a;
  int b;
};

struct Closed {
  int glist;     // arena list of units (reverse order) -- or -2 for a packed list
  int packed;    // index into packed_lists when glist == -2
  uint8_t kind;
  u64 qubits;
  int64_t cost;
  int prev;
};

struct St {
  std::vector<KD> ks;
  int64_t closed_cost = 0;
  int closed = -1;
  u64 h = 0;
};

struct Ctx {
  const CostModel &cm;
  const KernelizeOptions &o;
  int qmf, qms;
  u64 allq;
  std::vector<Node> arena;
  std::vector<Closed> closed;
  std::vector<std::vector<int>> packed_lists;

  Ctx(const CostModel &c, const KernelizeOptions &op, int n) : cm(c), o(op) {
    qmf = (o.kinds & 1) ? std::min(cm.q_max_fusion, o.L) : 0;
    qms = (o.kinds & 2) ? std::min(cm.q_max_shared, o.L) : -1;
    if (qms >= 0 && qms < 6) qms = -1;
    allq = n >= 64 ? ~0ull : ((1ull << n) - 1);
  }

  // lazy kind (reading R19): a kernel keeps every kind it still fits and is
  // charged the cheaper one (fusion on a tie) -- the two DP copies of
  // P:L1968 collapsed into one state
  int64_t kcost(u64 q, u64 a, int64_t g, int *kind) const {
    int64_t f = fits_fusion(q) ? cm.fusion_cost[popc(q) - 1] : INF64;
    int64_t sh = fits_shm(a) ? cm.alpha + g : INF64;
    if (kind) *kind = f <= sh ? K_FUSION : K_SHM;
    return std::min(f, sh);
  }
  int64_t cost(const KD &k) const { return kcost(k.qubits, k.active, k.gcost, nullptr); }
  bool feasible(u64 q, u64 a) const { return fits_fusion(q) || fits_shm(a); }
  bool fits_fusion(u64 q) const { return popc(q) >= 1 && popc(q) <= qmf; }
  bool fits_shm(u64 a) const { return qms >= 0 && popc(a | o.ls_set) <= qms; }
  // future summaries (set per position): qubits of the remaining units, the
  // non-insular qubits of the remaining units, and the qubits of remaining
  // units that are entirely insular
  u64 fut_q = ~0ull, fut_act = ~0ull, fut_diag = ~0ull;
  // a kernel is dead when no remaining unit could ever join it (Def. 5 via
  // the extensible sets); closing it then changes nothing but the state key
  bool dead(const KD &k) const {
    if (k.all) return false;
    if (o.lift) {
      if (k.extq & fut_act) return false;
      if ((k.extq | k.extins) & fut_diag) return false;
      return true;
    }
    return (k.extq & fut_q) == 0;
  }
  // may unit u join kernel k (Constraint 1 via extensible sets + size)?
  bool can_join(const KD &k, const Unit &u) const {
    if (!k.all) {
      if (o.lift) {
        const u64 ins = u.qubits & ~u.active;
        if (u.active & ~k.extq) return false;
        if (ins & ~(k.extins | k.extq)) return false;
      } else if (u.qubits & ~k.extq) {
        return false;
      }
    }
    return feasible(k.qubits | u.qubits, k.active | u.active);
  }
  u64 relevant(const KD &k, const Unit &u) const {
    u64 sh = k.qubits & u.qubits;
    return o.lift ? (sh & (k.active | u.active)) : sh;
  }
  int leaf(int unit) {
    arena.push_back(Node{unit, -2});
    return (int)arena.size() - 1;
  }
  int cat(int x, int y) {
    if (x < 0) return y;
    if (y < 0) return x;
    arena.push_back(Node{x, y});
    return (int)arena.size() - 1;
  }
  u64 hash(const St &s) const {
    u64 h = 1469598103934665603ull;
    auto mix = [&](u64 x) {
      h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    };
    for (const KD &k : s.ks) {
      mix(k.all ? 2 : 0);
      mix(k.qubits);
      mix(k.extq);
      mix(k.extins);
      mix(k.active);
      mix((u64)k.gcost);
    }
    return h;
  }
  // units of a kernel in ascending unit order: in-place additions append
  // increasing units and merged ALL kernels commute, so ascending order is a
  // valid internal order (Thm. dp-correct's in-kernel order)
  std::vector<int> units_of(int glist) const {
    std::vector<int> v, stack;
    if (glist >= 0) stack.push_back(glist);
    while (!stack.empty()) {
      int p = stack.back();
      stack.pop_back();
      if (arena[p].b == -2) {
        v.push_back(arena[p].a);
      } else {
        stack.push_back(arena[p].a);
        stack.push_back(arena[p].b);
      }
    }
    std::sort(v.begin(), v.end());
    return v;
  }
  // close the prefix of dead kernels; consecutive dead kernels are packed
  // with the post-processing rule first (the same packing the pruning
  // estimate assumes for them)
  void close_dead_prefix(St &s) {
    size_t d = 0;
    while (d < s.ks.size() && dead(s.ks[d])) d++;
    if (!d) return;
    std::vector<KD> pre(s.ks.begin(), s.ks.begin() + d);
    std::vector<std::vector<int>> groups;
    packed_cost(pre, &groups);
    for (auto &g : groups) {
      KD acc = pre[g[0]];
      for (size_t t = 1; t < g.size(); t++) {
        const KD &nx = pre[g[t]];
        acc.qubits |= nx.qubits;
        acc.active |= nx.active;
        acc.gcost += nx.gcost;
        acc.glist = cat(acc.glist, nx.glist);
      }
      int64_t c = cost(acc);
      int kd = 0;
      kcost(acc.qubits, acc.active, acc.gcost, &kd);
      closed.push_back(Closed{acc.glist, -1, (uint8_t)kd, acc.qubits, c, s.closed});
      s.closed = (int)closed.size() - 1;
      s.closed_cost += c;
    }
    s.ks.erase(s.ks.begin(), s.ks.begin() + d);
  }
  // post-processing: greedy packing of the open kernels in order
  int64_t packed_cost(const std::vector<KD> &ks, std::vector<std::vector<int>> *groups) const {
    int64_t total = 0;
    size_t i = 0;
    while (i < ks.size()) {
      KD cur = ks[i];
      std::vector<int> grp = {(int)i};
      size_t j = i + 1;
      while (j < ks.size()) {
        const KD &nx = ks[j];
        const u64 q = cur.qubits | nx.qubits, a = cur.active | nx.active;
        if (!feasible(q, a)) break;
        const int64_t merged = kcost(q, a, cur.gcost + nx.gcost, nullptr);
        if (merged > cost(cur) + cost(nx)) break;
        cur.qubits = q;
        cur.active = a;
        cur.gcost += nx.gcost;
        grp.push_back((int)j);
        j++;
      }
      total += cost(cur);
      if (groups) groups->push_back(grp);
      i = j;
    }
    return total;
  }
};

// attachment of single-qubit gates
std::vector<Unit> make_units(const std::vector<KGate> &seq, const CostModel &cm, bool attach) {
  const int m = (int)seq.size();
  std::vector<Unit> units;
  if (!attach) {
    for (int i = 0; i < m; i++) {
      Unit u;
      u.qubits = seq[i].qubits;
      u.active = seq[i].active;
      u.gcost = cm.gate_cost[seq[i].kind];
      u.gates = {i};
      units.push_back(u);
    }
    return units;
  }
  std::vector<int> host(m, -1);  // gate -> host gate index
  std::vector<int> after(m, 0);  // attached after the host?
  auto multi = [&](int i) { return popc(seq[i].qubits) > 1; };
  for (int i = 0; i < m; i++) {
    if (multi(i)) {
      host[i] = i;
      continue;
    }
    const u64 q = seq[i].qubits;
    int h = -1;
    for (int j = i + 1; j < m; j++)
      if (seq[j].qubits & q) {
        if (multi(j)) h = j;
        else continue;  // chain of single-qubit gates: keep looking for the successor host
        break;
      }
    if (h >= 0) {
      host[i] = h;
      continue;
    }
    for (int j = i - 1; j >= 0; j--)
      if (seq[j].qubits & q) {
        if (multi(j)) {
          h = j;
          break;
        }
      }
    if (h >= 0) {
      host[i] = h;
      after[i] = 1;
    }
  }
  // units in host order; standalone single-qubit gates with no host keep their place
  std::vector<int> unit_of(m, -1);
  for (int i = 0; i < m; i++) {
    if (host[i] == i || host[i] < 0) {
      unit_of[i] = (int)units.size();
      units.push_back(Unit{});
    }
  }
  for (int i = 0; i < m; i++)
    if (host[i] >= 0 && host[i] != i) unit_of[i] = unit_of[host[i]];
  // gates in execution order: attached-before (original order), host, attached-after
  std::vector<std::vector<int>> before(units.size()), aft(units.size());
  std::vector<int> hostg(units.size(), -1);
  for (int i = 0; i < m; i++) {
    int u = unit_of[i];
    if (host[i] == i || host[i] < 0) hostg[u] = i;
    else if (after[i]) aft[u].push_back(i);
    else before[u].push_back(i);
  }
  for (size_t u = 0; u < units.size(); u++) {
    Unit &U = units[u];
    for (int g : before[u]) U.gates.push_back(g);
    U.gates.push_back(hostg[u]);
    for (int g : aft[u]) U.gates.push_back(g);
    for (int g : U.gates) {
      U.qubits |= seq[g].qubits;
      U.active |= seq[g].active;
      U.gcost += cm.gate_cost[seq[g].kind];
    }
  }
  return units;
}

// exact commutation: two gates must keep their order iff they share a qubit
// that is not diagonal-type in both
bool order_is_valid(const std::vector<KGate> &seq, const std::vector<int> &order) {
  const int m = (int)seq.size();
  if ((int)order.size() != m) return false;
  std::vector<int> pos(m, -1);
  for (int p = 0; p < m; p++) {
    if (order[p] < 0 || order[p] >= m || pos[order[p]] >= 0) return false;
    pos[order[p]] = p;
  }
  for (int a = 0; a < m; a++)
    for (int b = a + 1; b < m; b++) {
      u64 sh = seq[a].qubits & seq[b].qubits;
      if (!sh) continue;
      if (!(sh & (seq[a].active | seq[b].active))) continue;
      if (pos[a] > pos[b]) return false;
    }
  return true;
}

}  // namespace

namespace {
KernelPlan dp_impl(const std::vector<KGate> &seq, const CostModel &cm, const KernelizeOptions &o,
                   bool dp_only);
}

KernelPlan dp_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                        const KernelizeOptions &o) {
  return dp_impl(seq, cm, o, false);
}

KernelPlan dp_only_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                             const KernelizeOptions &o) {
  return dp_impl(seq, cm, o, true);
}

namespace {
KernelPlan dp_impl(const std::vector<KGate> &seq, const CostModel &cm, const KernelizeOptions &o,
                   bool dp_only) {
  KernelPlan ordered = ordered_kernelize(seq, cm, o);
  if (getenv("ATLAS_DP_PARTNERS")) kMaxPartners = atoi(getenv("ATLAS_DP_PARTNERS"));
  if (getenv("ATLAS_DP_MERGES")) kMaxMergesPerGate = atoi(getenv("ATLAS_DP_MERGES"));
  const int m = (int)seq.size();
  if (m == 0) return ordered;
  std::vector<Unit> units = make_units(seq, cm, o.attach);
  const int nu = (int)units.size();
  int nq = 0;
  for (auto &g : seq) nq = std::max(nq, 64 - __builtin_clzll(g.qubits | 1));
  Ctx C(cm, o, nq);
  const int T = o.prune_T > 0 ? o.prune_T : INT_MAX;

  std::vector<u64> fq(nu + 1, 0), fa(nu + 1, 0), fd(nu + 1, 0);
  for (int i = nu - 1; i >= 0; i--) {
    fq[i] = fq[i + 1] | units[i].qubits;
    fa[i] = fa[i + 1] | units[i].active;
    fd[i] = fd[i + 1] | (units[i].active ? 0 : units[i].qubits);
  }
  std::vector<St> cur(1);
  // deterministic work budget (same on every rank, unlike a clock): when the
  // DP would exceed it, Kernelize falls back to the cheaper of the front
  // packing and OrderedKernelize (R29)
  long long emitted = 0;
  const long long budget = (o.dp_budget > 0 && !dp_only) ? o.dp_budget : LLONG_MAX;
  auto fallback = [&]() {
    KernelPlan best_plan = ordered;
    if (o.front) {
      KernelPlan fr = front_kernelize(seq, cm, o);
      std::vector<int> ford;
      for (auto &K : fr.kernels) ford.insert(ford.end(), K.gates.begin(), K.gates.end());
      if (order_is_valid(seq, ford) && fr.total < best_plan.total) best_plan = fr;
    }
    return best_plan;
  };
  // branch and bound: the cheaper of the front packing and OrderedKernelize
  // is computed first; a DP state whose closed kernels alone already cost
  // more can never be returned (the DP result is taken only when <= it), so
  // it is dropped.  If every state is dropped the DP cannot win.
  const KernelPlan ub_plan = dp_only ? KernelPlan{} : fallback();
  const int64_t UB = (getenv("ATLAS_DP_NOBOUND") || dp_only) ? INF64 : ub_plan.total;
  for (int i = 0; i < nu; i++) {
    if (emitted > budget) {
      if (getenv("ATLAS_DEBUG")) fprintf(stderr, "[kernelize] units=%d budget out at %d ub=%lld\n", nu, i, (long long)UB);
      return ub_plan;
    }
    const Unit &u = units[i];
    if (!getenv("ATLAS_DP_NOFUT")) {
      C.fut_q = fq[i + 1];
      C.fut_act = fa[i + 1];
      C.fut_diag = fd[i + 1];
    }
    // ---- pruning at the beginning of the iteration
    if ((int)cur.size() >= T) {
      std::vector<std::pair<int64_t, int>> sc;
      for (int s = 0; s < (int)cur.size(); s++)
        sc.push_back({cur[s].closed_cost + C.packed_cost(cur[s].ks, nullptr), s});
      std::sort(sc.begin(), sc.end(), [&](const auto &a, const auto &b) {
        if (a.first != b.first) return a.first < b.first;
        return cur[a.second].h < cur[b.second].h;
      });
      std::vector<St> keep;
      for (int k = 0; k < std::max(1, T / 2); k++) keep.push_back(std::move(cur[sc[k].second]));
      cur.swap(keep);
    }
    std::vector<St> next;
    std::unordered_map<u64, std::vector<int>> idx;
    auto emit = [&](St &&s) {
      emitted++;
      C.close_dead_prefix(s);
      if (s.closed_cost > UB) return;
      if ((int)next.size() >= 8 * T && T < INT_MAX / 16) {
        // keep the working set bounded inside an iteration as well (same
        // criterion as the pruning of P:L2496)
        std::vector<std::pair<int64_t, int>> sc;
        for (int q = 0; q < (int)next.size(); q++)
          sc.push_back({next[q].closed_cost + C.packed_cost(next[q].ks, nullptr), q});
        std::sort(sc.begin(), sc.end());
        std::vector<St> keep;
        for (int q = 0; q < T; q++) keep.push_back(std::move(next[sc[q].second]));
        next.swap(keep);
        idx.clear();
        for (int q = 0; q < (int)next.size(); q++) idx[next[q].h].push_back(q);
      }
      s.h = C.hash(s);
      auto &bucket = idx[s.h];
      for (int j : bucket) {
        if (next[j].ks == s.ks) {
          if (s.closed_cost < next[j].closed_cost) next[j] = std::move(s);
          return;
        }
      }
      bucket.push_back((int)next.size());
      next.push_back(std::move(s));
    };
    // ExtQ maintenance (Alg. ExtQ) for every kernel except the host `hk`;
    // kernels that lose ALL may merge with another ALL kernel (deferral).
    // Produces all resulting states.
    // ExtQ maintenance (Alg. ExtQ) for every kernel except the
    // host `hk` (the kernel now holding C[i]).  A kernel K' with ExtQ = ALL
    // that C[i] touches loses ALL; with deferred merging
    // it may instead be merged with another ALL kernel -- with
    // the host itself (that is how a gate joins a still-floating kernel; the
    // merged kernel keeps ExtQ = ALL) or, at most once per gate, with another
    // ALL kernel (the merge then loses ALL).
    std::function<void(St &, int, size_t, bool, int)> update;
    update = [&](St &s, int hk, size_t j, bool may_merge, int budget) {
      for (; j < s.ks.size(); j++) {
        if ((int)j == hk) continue;
        KD &k = s.ks[j];
        if (!k.all) {
          k.extq &= ~u.qubits;
          k.extins &= ~u.qubits;
          continue;
        }
        if (!C.relevant(k, u)) continue;
        int nonhost = 0;
        for (int pp = (int)s.ks.size() - 1; pp >= 0; pp--) {
          const size_t p = (size_t)pp;
          if (p == j) continue;
          const KD &q = s.ks[p];
          if (!q.all) continue;
          const bool with_host = (int)p == hk;
          if (budget <= 0) continue;
          if (!with_host && (!may_merge || nonhost >= kMaxPartners)) continue;
          if (!with_host) nonhost++;
          const int at = (int)std::max(p, j);
          if (!with_host && hk >= 0 && at > hk) continue;
          if (!C.feasible(k.qubits | q.qubits, k.active | q.active)) continue;
          St s2 = s;
          const KD &a = s2.ks[j];
          const KD &b = s2.ks[p];
          KD mg = a;
          mg.qubits |= b.qubits;
          mg.active |= b.active;
          mg.gcost += b.gcost;
          mg.glist = C.cat(a.glist, b.glist);
          mg.nunits = a.nunits + b.nunits;
          if (with_host) {
            mg.all = true;  // C[i] is inside: nothing outside touched it
          } else {
            mg.all = false;
            mg.extq = mg.qubits & ~u.qubits;
            mg.extins = C.allq & ~u.qubits;
          }
          const int rm = (int)std::min(p, j);
          s2.ks[at] = mg;
          s2.ks.erase(s2.ks.begin() + rm);
          int hk2 = with_host ? at - 1 : (hk > rm ? hk - 1 : hk);
          update(s2, hk2, (size_t)rm, with_host ? may_merge : false, budget - 1);
        }
        k.all = false;
        k.extq = k.qubits & ~u.qubits;
        k.extins = C.allq & ~u.qubits;
      }
      emit(std::move(s));
    };

    // greedy deferred merging: every ALL kernel of the host's kind that C[i]
    // touches is merged into the host while it fits (one extra branch)
    auto merge_all = [&](St &s, int hk) {
      if (!s.ks[hk].all) return;
      int merged = 0;
      for (int j = 0; j < (int)s.ks.size(); j++) {
        if (j == hk) continue;
        KD &k = s.ks[j];
        if (!k.all || !C.relevant(k, u)) continue;
        KD &h = s.ks[hk];
        if (!C.feasible(k.qubits | h.qubits, k.active | h.active)) continue;
        if (j > hk) continue;
        h.qubits |= k.qubits;
        h.active |= k.active;
        h.gcost += k.gcost;
        h.glist = C.cat(k.glist, h.glist);
        h.nunits += k.nunits;
        s.ks.erase(s.ks.begin() + j);
        hk--;
        j--;
        merged++;
      }
      if (merged < 2) return;  // single merges are covered by update()
      update(s, hk, 0, false, 0);
    };

    // deferred merging, greedy group branch: the ALL kernels that C[i] makes
    // lose ALL are packed together (in order, same kind, while they fit)
    // before they are restricted -- the "merge with the other ALL kernels"
    // of P:L2480-2482 applied to all of them at once
    auto merge_group = [&](St &s, int hk) {
      std::vector<int> J;
      for (int j = 0; j < (int)s.ks.size(); j++) {
        if (j == hk || !s.ks[j].all) continue;
        if (C.relevant(s.ks[j], u)) J.push_back(j);
      }
      if (J.size() < 2) return;
      std::vector<char> erase(s.ks.size(), 0);
      bool any = false;
      size_t a = 0;
      while (a < J.size()) {
        KD acc = s.ks[J[a]];
        size_t b = a + 1;
        int last = J[a];
        while (b < J.size()) {
          const KD &nx = s.ks[J[b]];
          if (!C.feasible(acc.qubits | nx.qubits, acc.active | nx.active)) break;
          acc.qubits |= nx.qubits;
          acc.active |= nx.active;
          acc.gcost += nx.gcost;
          acc.glist = C.cat(acc.glist, nx.glist);
          acc.nunits += nx.nunits;
          erase[last] = 1;
          last = J[b];
          b++;
        }
        if (b - a >= 2) {
          s.ks[last] = acc;
          any = true;
        }
        a = b;
      }
      if (!any) return;
      std::vector<KD> ks2;
      int hk2 = -1;
      for (int j = 0; j < (int)s.ks.size(); j++) {
        if (erase[j]) continue;
        if (j == hk) hk2 = (int)ks2.size();
        ks2.push_back(s.ks[j]);
      }
      s.ks.swap(ks2);
      update(s, hk2, 0, false, 0);
    };

    for (St &s : cur) {
      // a gate joining an open kernel K in place must not conflict with any
      // kernel ordered after K (with the insular lifting, kernels that only
      // share insular qubits may have been ordered after K)
      std::vector<char> later_conflict(s.ks.size() + 1, 0);
      for (int j = (int)s.ks.size() - 1; j >= 0; j--) {
        const KD &k = s.ks[j];
        const u64 sh = k.qubits & u.qubits;
        const bool cf = o.lift ? (sh & (k.active | u.active)) != 0 : sh != 0;
        later_conflict[j] = later_conflict[j + 1] || cf;
      }
      auto in_place_ok = [&](int j) { return s.ks[j].all || !later_conflict[j + 1]; };
      // subsumption: nested qubit sets and allowed -> add directly, no branching
      int sub = -1;
      for (size_t j = 0; j < s.ks.size(); j++) {
        const KD &k = s.ks[j];
        bool nested = (u.qubits & ~k.qubits) == 0 || (k.qubits & ~u.qubits) == 0;
        if (nested && C.can_join(k, u) && in_place_ok((int)j)) {
          sub = (int)j;
          break;
        }
      }
      // a purely diagonal unit (every qubit insular) commutes with everything
      // except non-insular uses of its qubits: with the lifting it joins the
      // most recent open kernel that may take it instead of floating as an
      // ALL singleton (reading R20)
      if (sub < 0 && o.lift && u.active == 0) {
        for (int j = (int)s.ks.size() - 1; j >= 0; j--)
          if (C.can_join(s.ks[j], u) && in_place_ok(j)) {
            sub = j;
            break;
          }
      }
      std::vector<int> targets;
      if (sub >= 0) {
        targets.push_back(sub);
      } else {
        for (size_t j = 0; j < s.ks.size(); j++)
          if (!s.ks[j].all && C.can_join(s.ks[j], u) && in_place_ok((int)j)) targets.push_back((int)j);
      }
      for (int j : targets) {
        St s2 = s;
        KD k = s2.ks[j];
        k.qubits |= u.qubits;
        k.active |= u.active;
        k.gcost += u.gcost;
        k.glist = C.cat(k.glist, C.leaf(i));
        k.nunits++;
        int hk = j;
        if (k.all) {  // monotonicity does not apply: move K to the end
          s2.ks.erase(s2.ks.begin() + j);
          s2.ks.push_back(k);
          hk = (int)s2.ks.size() - 1;
        } else {
          s2.ks[j] = k;
        }
        St s3 = s2, s4 = s2;
        update(s2, hk, 0, true, kMaxMergesPerGate);
        merge_all(s3, hk);
        merge_group(s4, hk);
      }
      if (sub >= 0) continue;
      // new singleton kernel at the end (lazy kind, see kcost)
      if (C.feasible(u.qubits, u.active)) {
        St s2 = s;
        KD k;
        k.all = true;
        k.qubits = u.qubits;
        k.active = u.active;
        k.gcost = u.gcost;
        k.glist = C.leaf(i);
        k.nunits = 1;
        s2.ks.push_back(k);
        St s3 = s2, s4 = s2;
        update(s2, (int)s2.ks.size() - 1, 0, true, kMaxMergesPerGate);
        merge_all(s3, (int)s3.ks.size() - 1);
        merge_group(s4, (int)s4.ks.size() - 1);
      }
    }
    if (next.empty()) {
      if (getenv("ATLAS_DEBUG")) fprintf(stderr, "[kernelize] units=%d bounded out at %d emitted %lld\n", nu, i, (long long)emitted);
      if (UB < INF64) return ub_plan;  // every state is bounded out
      fail(ATLAS_E_INFEASIBLE, "Kernelize: unit %d fits no kernel", i);
    }
    if (getenv("ATLAS_DEBUG_DP"))
    {
      size_t tot = 0, mx = 0;
      for (auto &x : next) { tot += x.ks.size(); mx = std::max(mx, x.ks.size()); }
      fprintf(stderr, "[dp] unit %d/%d states %zu -> %zu arena %zu open avg %.1f max %zu\n", i, nu, cur.size(), next.size(), C.arena.size(), (double)tot / next.size(), mx);
    }
    cur.swap(next);
  }
  // ---- DP_best = min_KS DP[|C|, KS] + Cost(KS), with post-processing
  int best = -1;
  int64_t best_cost = INF64;
  for (int s = 0; s < (int)cur.size(); s++) {
    int64_t c = cur[s].closed_cost + C.packed_cost(cur[s].ks, nullptr);
    if (c < best_cost || (c == best_cost && cur[s].h < cur[best].h)) {
      best_cost = c;
      best = s;
    }
  }
  const St &B = cur[best];
  // reconstruct: closed kernels (closing order), then the packed open kernels
  struct Out {
    std::vector<int> units;
    int kind;
  };
  std::vector<Out> outs;
  {
    std::vector<int> chain;
    for (int c = B.closed; c >= 0; c = C.closed[c].prev) chain.push_back(c);
    std::reverse(chain.begin(), chain.end());
    for (int c : chain) outs.push_back(Out{C.units_of(C.closed[c].glist), C.closed[c].kind});
    std::vector<std::vector<int>> groups;
    C.packed_cost(B.ks, &groups);
    for (auto &g : groups) {
      Out o2{{}, 0};
      for (int j : g) {
        auto us = C.units_of(B.ks[j].glist);
        o2.units.insert(o2.units.end(), us.begin(), us.end());
      }
      outs.push_back(o2);
    }
  }
  KernelPlan kp;
  std::vector<int> order;
  for (auto &ot : outs) {
    Kernel K;
    u64 q = 0, act = o.ls_set;
    int64_t gs = 0;
    for (int ui : ot.units)
      for (int g : units[ui].gates) {
        K.gates.push_back(g);
        order.push_back(g);
        q |= seq[g].qubits;
        act |= seq[g].active;
        gs += cm.gate_cost[seq[g].kind];
      }
    int kd = 0;
    K.cost = C.kcost(q, act, gs, &kd);
    K.kind = kd;
    K.qubits = K.kind == K_FUSION ? q : act;
    kp.total += K.cost;
    kp.kernels.push_back(K);
  }
  const bool valid = order_is_valid(seq, order);
  if (getenv("ATLAS_DEBUG"))
    fprintf(stderr, "[kernelize] units=%d dp_cost=%lld kernels=%zu ordered=%lld (%zu) valid=%d arena=%zu\n",
            nu, (long long)kp.total, kp.kernels.size(), (long long)ordered.total,
            ordered.kernels.size(), (int)valid, C.arena.size());
  if (getenv("ATLAS_DEBUG_KEEP") || dp_only) return kp;
  // the cheapest valid candidate: the DP, OrderedKernelize (Thm. dp-optimal
  // guarantees DP <= Ordered without pruning; pruning may worsen
  // it) and the commutation-aware front packing (R29)
  KernelPlan best_plan = ub_plan;
  if (valid && kp.total <= best_plan.total) best_plan = kp;
  return best_plan;
}

}  // namespace

}  // namespace atlas
