// staging.cpp -- circuit staging (PAPER.md §"Circuit Staging").
//
// The paper solves a binary ILP (objective P:L1491, constraints c1-c6
// P:L1495-1502) with PuLP+HiGHS for s = 1, 2, ... and returns the first
// feasible s (Alg. Stage; Thm. ilp-optimal).  No ILP
// solver exists in this image, so we solve the same problem exactly by search:
//
//  * For fixed per-stage (local, global) sets the objective does not depend on
//    F, and the maximal F (every gate finishes in the first stage where c3 and
//    c4 allow) is feasible whenever any F is (SURVEY §8c O2 lemma, pinned in
//    tests/test_oracle_planner.py against a literal ILP enumeration).  So the
//    ILP reduces to a search over sequences of global sets with maximal
//    execution; gate stage = min{k : F_{g,k} = 1}.
//  * R = 0 on one NVSwitch box (R7): A_{q,k} + B_{q,k} = 1, so the
//    objective (Eq. P:L1477) is (1 + c) * sum_k |G_k \ G_{k-1}|.
//  * Search: layered DP over states (executed-gate frontier, current global
//    set); per state keep the minimum cost and the lexicographically smallest
//    prefix of global bitmasks (canonical tie-break, R5).  A layer
//    is expanded only with transitions that execute at least one new gate
//    (a stage without progress never appears in a minimum-s solution).  The
//    final stage is solved in closed form: its global set must avoid every
//    non-insular qubit of the remaining gates; the cheapest such set keeps
//    all still-allowed previous globals and fills with the lowest qubits.
//  * Budget: when a layer would exceed the state budget the layer is cut to
//    the best states (most gates executed, then cost) and the plan is marked
//    exact = false (reported in the plan JSON and DESIGN.md).
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "internal.h"

namespace atlas {

namespace {

struct Frontier {
  std::vector<u64> w;
  bool operator==(const Frontier &o) const { return w == o.w; }
};

struct StateKey {
  u64 h;
  u64 g;
  bool operator==(const StateKey &o) const { return h == o.h && g == o.g; }
};
struct KeyHash {
  size_t operator()(const StateKey &k) const { return (size_t)(k.h * 0x9E3779B97F4A7C15ull ^ k.g); }
};

struct State {
  Frontier f;
  u64 g;
  double cost;
  std::vector<u64> prefix;
  int ndone;
};

struct Ctx {
  int n, L, G, m;
  const std::vector<GateInfo> *info;
  std::vector<std::vector<int>> preds;
  long evals = 0;

  bool done(const Frontier &f, int g) const { return (f.w[g >> 6] >> (g & 63)) & 1; }
  void set(Frontier &f, int g) const { f.w[g >> 6] |= 1ull << (g & 63); }

  // maximal execution of one stage with local set `loc` (c3, c4)
  int maxexec(Frontier &f, u64 loc) {
    evals++;
    int added = 0;
    for (int g = 0; g < m; g++) {
      if (done(f, g)) continue;
      if ((*info)[g].nonins & ~loc) continue;
      bool ok = true;
      for (int p : preds[g])
        if (!done(f, p)) { ok = false; break; }
      if (ok) { set(f, g); added++; }
    }
    return added;
  }
  u64 remaining_nonins(const Frontier &f) const {
    u64 u = 0;
    for (int g = 0; g < m; g++)
      if (!done(f, g)) u |= (*info)[g].nonins;
    return u;
  }
  u64 hash(const Frontier &f) const {
    u64 h = 1469598103934665603ull;
    for (u64 x : f.w) { h ^= x; h *= 1099511628211ull; h ^= h >> 29; }
    return h;
  }
};

u64 full_mask(int n) { return n == 64 ? ~0ull : ((1ull << n) - 1); }

// lowest-index completion: keep prev ∩ allowed, fill with the lowest allowed qubits
u64 final_global(u64 prev, u64 allowed, int G) {
  u64 g = prev & allowed;
  int need = G - popc(g);
  u64 rest = allowed & ~g;
  while (need > 0 && rest) {
    u64 lo = rest & (~rest + 1);
    g |= lo;
    rest ^= lo;
    need--;
  }
  return need == 0 ? g : ~0ull;
}

bool better(double c1, const std::vector<u64> &p1, double c2, const std::vector<u64> &p2) {
  if (c1 != c2) return c1 < c2;
  return p1 < p2;
}

}  // namespace

StagePlan stage_circuit(int n, int L, int G, const std::vector<GateInfo> &info, int s_max,
                        double c, long budget) {
  const int m = (int)info.size();
  for (int g = 0; g < m; g++)
    if (popc(info[g].nonins) > L)
      fail(ATLAS_E_INFEASIBLE, "gate %d has %d non-insular qubits > L = %d", g,
           popc(info[g].nonins), L);
  StagePlan sp;
  const u64 all = full_mask(n);
  if (G == 0 || m == 0) {
    // with no global qubit every gate is local: one stage, cost 0
    u64 g0 = 0;
    if (G > 0) {
      u64 u = 0;
      for (auto &x : info) u |= x.nonins;
      g0 = final_global(0, all & ~u, G);
    }
    sp.s = 1;
    sp.local = {all & ~g0};
    sp.global = {g0};
    sp.gate_stage.assign(m, 0);
    return sp;
  }
  Ctx C{n, L, G, m, &info, {}, 0};
  C.preds.resize(m);
  {
    std::vector<int> last(n, -1);
    for (int g = 0; g < m; g++) {
      u64 q = info[g].qmask;
      while (q) {
        int b = ctz(q);
        q &= q - 1;
        if (last[b] >= 0 &&
            std::find(C.preds[g].begin(), C.preds[g].end(), last[b]) == C.preds[g].end())
          C.preds[g].push_back(last[b]);  // edge set E: adjacent pairs
        last[b] = g;
      }
    }
  }
  // candidate global sets in increasing bitmask order (Gosper)
  std::vector<u64> cand;
  {
    u64 v = (1ull << G) - 1;
    while (v <= all && v != 0) {
      cand.push_back(v);
      u64 t = v | (v - 1);
      if (t == ~0ull) break;
      v = (t + 1) | (((~t & -~t) - 1) >> (ctz(v) + 1));
    }
  }
  const int words = (m + 63) / 64;
  const double unit = 1.0 + c;
  bool exact = true;

  // s = 1
  {
    u64 u = 0;
    for (auto &x : info) u |= x.nonins;
    u64 g0 = final_global(0, all & ~u, G);
    if (g0 != ~0ull) {
      sp.s = 1;
      sp.local = {all & ~g0};
      sp.global = {g0};
      sp.gate_stage.assign(m, 0);
      return sp;
    }
  }
  // layer 0
  std::vector<State> layer;
  {
    std::unordered_map<StateKey, int, KeyHash> idx;
    for (u64 g0 : cand) {
      Frontier f{std::vector<u64>(words, 0)};
      int a = C.maxexec(f, all & ~g0);
      if (a == 0) continue;
      StateKey k{C.hash(f), g0};
      if (idx.count(k)) continue;
      idx[k] = (int)layer.size();
      layer.push_back(State{f, g0, 0.0, {g0}, a});
    }
  }
  for (int s = 2; s <= s_max; s++) {
    // completion in one more stage?
    int best = -1;
    double best_cost = 0;
    std::vector<u64> best_pref;
    for (int i = 0; i < (int)layer.size(); i++) {
      const State &st = layer[i];
      u64 u = C.remaining_nonins(st.f);
      u64 gl = final_global(st.g, all & ~u, G);
      if (gl == ~0ull) continue;
      double cost = st.cost + unit * popc(gl & ~st.g);
      std::vector<u64> pref = st.prefix;
      pref.push_back(gl);
      if (best < 0 || better(cost, pref, best_cost, best_pref)) {
        best = i;
        best_cost = cost;
        best_pref = pref;
      }
    }
    if (best >= 0) {
      sp.s = s;
      sp.cost = best_cost;
      sp.exact = exact;
      sp.global = best_pref;
      for (u64 g : sp.global) sp.local.push_back(all & ~g);
      // replay maximal execution to assign gate stages
      Frontier f{std::vector<u64>(words, 0)};
      sp.gate_stage.assign(m, -1);
      for (int k = 0; k < s; k++) {
        Frontier before = f;
        C.maxexec(f, sp.local[k]);
        for (int g = 0; g < m; g++)
          if (C.done(f, g) && !C.done(before, g)) sp.gate_stage[g] = k;
      }
      for (int g = 0; g < m; g++)
        if (sp.gate_stage[g] < 0) fail(ATLAS_E_INFEASIBLE, "internal: staging replay incomplete");
      sp.states_explored = C.evals;
      return sp;
    }
    if (s == s_max) break;
    // expand to the next layer
    std::vector<State> next;
    std::unordered_map<StateKey, int, KeyHash> idx;
    long projected = (long)layer.size() * (long)cand.size();
    if (projected > budget) {
      // keep the states that executed the most gates (then cheapest, then lexicographic)
      std::sort(layer.begin(), layer.end(), [](const State &a, const State &b) {
        if (a.ndone != b.ndone) return a.ndone > b.ndone;
        if (a.cost != b.cost) return a.cost < b.cost;
        return a.prefix < b.prefix;
      });
      size_t keep = std::max<size_t>(1, (size_t)(budget / (long)cand.size()));
      if (layer.size() > keep) {
        layer.resize(keep);
        exact = false;
      }
    }
    for (const State &st : layer) {
      for (u64 g : cand) {
        Frontier f = st.f;
        int a = C.maxexec(f, all & ~g);
        if (a == 0) continue;
        double cost = st.cost + unit * popc(g & ~st.g);
        StateKey k{C.hash(f), g};
        auto it = idx.find(k);
        std::vector<u64> pref = st.prefix;
        pref.push_back(g);
        if (it == idx.end()) {
          idx[k] = (int)next.size();
          next.push_back(State{f, g, cost, pref, st.ndone + a});
        } else if (better(cost, pref, next[it->second].cost, next[it->second].prefix)) {
          next[it->second].cost = cost;
          next[it->second].prefix = pref;
        }
      }
    }
    layer.swap(next);
    if (layer.empty()) break;
  }
  fail(ATLAS_E_INFEASIBLE, "no staging with at most %d stages", s_max);
}

}  // namespace atlas
