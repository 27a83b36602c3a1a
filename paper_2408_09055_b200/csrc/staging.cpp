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
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

#include "internal.h"

namespace atlas {

namespace {

typedef std::vector<u64> Frontier;

struct FHash {
  size_t operator()(const Frontier &f) const {
    u64 h = 1469598103934665603ull;
    for (u64 x : f) { h ^= x; h *= 1099511628211ull; h ^= h >> 29; }
    return (size_t)h;
  }
};

bool subset(const Frontier &a, const Frontier &b) {  // a ⊆ b
  for (size_t i = 0; i < a.size(); i++)
    if (a[i] & ~b[i]) return false;
  return true;
}

int fcount(const Frontier &f) {
  int c = 0;
  for (u64 x : f) c += popc(x);
  return c;
}

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

// all subsets of `pool` with exactly k bits, ascending as integers
void combos(u64 pool, int k, std::vector<u64> &out) {
  out.clear();
  std::vector<int> bits;
  for (u64 p = pool; p; p &= p - 1) bits.push_back(ctz(p));
  const int nb = (int)bits.size();
  if (k > nb || k < 0) return;
  if (k == 0) {
    out.push_back(0);
    return;
  }
  std::vector<int> idx(k);
  for (int i = 0; i < k; i++) idx[i] = i;
  for (;;) {
    u64 v = 0;
    for (int i = 0; i < k; i++) v |= 1ull << bits[idx[i]];
    out.push_back(v);
    int i = k - 1;
    while (i >= 0 && idx[i] == nb - k + i) i--;
    if (i < 0) break;
    idx[i]++;
    for (int j = i + 1; j < k; j++) idx[j] = idx[j - 1] + 1;
  }
  std::sort(out.begin(), out.end());
}

struct Search {
  int n, L, G, m, words;
  u64 all;
  const std::vector<GateInfo> *info;
  std::vector<std::vector<int>> preds, succs;
  long evals = 0;
  long budget;
  bool over = false;
  bool dbg = getenv("ATLAS_DEBUG_STAGE") != nullptr;
  // scratch of levels()
  std::vector<int> lv;
  std::vector<u64> lw;

  bool done(const Frontier &f, int g) const { return (f[g >> 6] >> (g & 63)) & 1; }

  // maximal execution of one stage with local set `loc` (c3, c4): one pass in
  // circuit order reaches the fixpoint, since every predecessor comes earlier
  int maxexec(Frontier &f, u64 loc) {
    evals++;
    int added = 0;
    for (int g = 0; g < m; g++) {
      if (done(f, g)) continue;
      if ((*info)[g].nonins & ~loc) continue;
      bool ok = true;
      for (int p : preds[g])
        if (!done(f, p)) { ok = false; break; }
      if (ok) { f[g >> 6] |= 1ull << (g & 63); added++; }
    }
    return added;
  }
  u64 remaining_nonins(const Frontier &f) const {
    u64 u = 0;
    for (int g = 0; g < m; g++)
      if (!done(f, g)) u |= (*info)[g].nonins;
    return u;
  }

  // Stage levels of the remaining gates (lower bounds, exact reasoning):
  // forward h(g) = earliest stage (0 = the next one) any plan can run g in.
  // With H = max h over g's pending predecessors, every pending ancestor a
  // of g with h(a) = H runs no earlier than H and no later than g, so if g
  // ran at H all of them would share that stage and the union W of their
  // non-insular qubits would have to be local: |W| > L forces h(g) = H + 1.
  // Backward b(g) = stages any plan needs after g's stage, by the mirror
  // argument over descendants.  Returns the lower bound on the number of
  // stages that finish every pending gate (a virtual sink after all of
  // them); fills fwd (h) and bwd (b) per gate (-1 = done).
  int levels(const Frontier &f, std::vector<int> &fwd, std::vector<int> &bwd) {
    fwd.assign(m, -1);
    bwd.assign(m, -1);
    lw.assign(m, 0);
    int top = -1;
    for (int g = 0; g < m; g++) {
      if (done(f, g)) continue;
      int H = 0;
      for (int p : preds[g])
        if (!done(f, p)) H = std::max(H, fwd[p]);
      u64 W = (*info)[g].nonins;
      for (int p : preds[g])
        if (!done(f, p) && fwd[p] == H) W |= lw[p];
      if (popc(W) > L) { H++; W = (*info)[g].nonins; }
      fwd[g] = H;
      lw[g] = W;
      top = std::max(top, H);
    }
    if (top < 0) return 0;
    u64 Ws = 0;
    for (int g = 0; g < m; g++)
      if (fwd[g] == top) Ws |= lw[g];
    const int lb = popc(Ws) > L ? top + 2 : top + 1;
    lw.assign(m, 0);
    for (int g = m - 1; g >= 0; g--) {
      if (done(f, g)) continue;
      int B = 0;
      for (int q : succs[g]) B = std::max(B, bwd[q]);
      u64 V = (*info)[g].nonins;
      for (int q : succs[g])
        if (bwd[q] == B) V |= lw[q];
      if (popc(V) > L) { B++; V = (*info)[g].nonins; }
      bwd[g] = B;
      lw[g] = V;
    }
    return lb;
  }
};

struct MemoKey {
  Frontier f;
  u64 g, b;
  int k;
  bool operator==(const MemoKey &o) const { return g == o.g && b == o.b && k == o.k && f == o.f; }
};
struct MemoHash {
  size_t operator()(const MemoKey &x) const {
    return FHash()(x.f) ^ (size_t)(x.g * 0x9E3779B97F4A7C15ull) ^ (size_t)(x.b * 0xC2B2AE3D27D4EB4Full) ^
           (size_t)x.k;
  }
};

// global set of the next stage for a chosen constrained part: keep the
// free previous globals (cost 0; the lowest ones if there are more than the
// free slots), then the lowest other free qubits -- free qubits are
// interchangeable for every later stage, so this is the cheapest and then
// lexicographically smallest completion (R5)
u64 fill_free(u64 c, u64 prev, u64 freeq, int G, u64 prevb = 0) {
  int need = G - popc(c);
  u64 g = c;
  // with regional qubits: previous globals first (no global update either)
  for (u64 p = prevb & freeq; p && need > 0; p &= p - 1) { g |= p & (~p + 1); need--; }
  for (u64 p = prev & freeq & ~g; p && need > 0; p &= p - 1) { g |= p & (~p + 1); need--; }
  for (u64 p = freeq & ~g; p && need > 0; p &= p - 1) { g |= p & (~p + 1); need--; }
  return need == 0 ? g : ~0ull;
}

}  // namespace

StagePlan stage_circuit(int n, int L, int G, const std::vector<GateInfo> &info, int s_max,
                        double c, long budget, int R) {
  // G = non-local qubits (the rank bits); R of them are regional and
  // Gg = G - R global (the paper's three tiers, Def. P:L1405-1417; R = 0 on
  // one NVSwitch box, R > 0 emulates a two-tier interconnect, R7)
  const int Gg = G - R;
  const int m = (int)info.size();
  for (int g = 0; g < m; g++)
    if (popc(info[g].nonins) > L)
      fail(ATLAS_E_INFEASIBLE, "gate %d has %d non-insular qubits > L = %d", g,
           popc(info[g].nonins), L);
  StagePlan sp;
  const u64 all = full_mask(n);
  {
    // one stage: the global set avoids every non-insular qubit (cost 0)
    u64 u = 0;
    for (auto &x : info) u |= x.nonins;
    const u64 g0 = G == 0 ? 0 : final_global(0, all & ~u, G);
    if (g0 != ~0ull) {
      u64 b0 = 0;
      for (u64 p = g0; p && popc(b0) < Gg; p &= p - 1) b0 |= p & (~p + 1);
      sp.s = 1;
      sp.local = {all & ~g0};
      sp.global = {b0};
      sp.gate_stage.assign(m, 0);
      return sp;
    }
  }
  Search S;
  S.n = n; S.L = L; S.G = G; S.m = m; S.words = (m + 63) / 64; S.all = all;
  S.info = &info; S.budget = std::max(1000L, budget);
  S.preds.resize(m);
  S.succs.resize(m);
  {
    std::vector<int> last(n, -1);
    for (int g = 0; g < m; g++) {
      u64 q = info[g].qmask;
      while (q) {
        int b = ctz(q);
        q &= q - 1;
        if (last[b] >= 0 &&
            std::find(S.preds[g].begin(), S.preds[g].end(), last[b]) == S.preds[g].end()) {
          S.preds[g].push_back(last[b]);  // edge set E: adjacent pairs
          S.succs[last[b]].push_back(g);
        }
        last[b] = g;
      }
    }
  }
  const double unit = 1.0 + c;  // R = 0: every swap updates a local and a global qubit
  // the objective (Eq. P:L1491): newly local qubits + c * newly global ones
  auto step_cost = [&](u64 g, u64 b, u64 g2, u64 b2) {
    return R == 0 ? unit * popc(g2 & ~g) : (double)popc(g & ~g2) + c * popc(b2 & ~b);
  };
  // all global subsets of a non-local set (ascending); R = 0: the set itself
  auto global_subsets = [&](u64 g2, std::vector<u64> &out) {
    out.clear();
    if (R == 0) {
      out.push_back(g2);
      return;
    }
    combos(g2, Gg, out);
  };
  const Frontier empty(S.words, 0);
  // Depth-first branch and bound over the per-stage global sets, in
  // increasing bitmask order (so among plans of equal cost the first found
  // is the canonical one, R5), for s = the level lower bound,
  // s + 1, ...  (Thm. ilp-optimal: the minimum s first; then the
  // minimum objective Eq. P:L1477).  Every pruning is exact:
  //  * viability: the stage-level bound of the remaining gates must fit the
  //    stages left;
  //  * cost bound: cost so far + unit * (current globals that some remaining
  //    gate forces local at the next stage + for every later boundary the
  //    globals that cannot avoid such a gate) >= the best plan found;
  //  * transpositions: a (frontier, global set, stage) reached again at no
  //    lower cost (a later, lexicographically larger prefix);
  //  * global sets differ only in their constrained part (qubits with
  //    remaining non-insular gates); the free qubits are completed by
  //    fill_free.
  std::vector<int> fwd, bwd;
  std::vector<u64> cons_sets;
  bool exact = true;
  int sfound = -1;
  double best_cost = 1e300;
  std::vector<u64> best_pref, best_bpref;
  auto lower_cost = [&](int s, int k, u64 g, u64 b, const std::vector<int> &fw, const std::vector<int> &bw) {
    // k = index of the stage just executed with global set g
    std::vector<u64> F(s + 1, 0);  // F[j]: qubits forced local at stage j+1 if global at j
    for (int x = 0; x < m; x++) {
      if (fw[x] < 0) continue;
      const int e = k + 1 + fw[x], lat = s - 1 - bw[x];
      const u64 nq = info[x].nonins;
      if (lat <= k + 1) F[k] |= nq;
      for (int j = k + 1; j <= s - 2; j++)
        if (e >= j && lat <= j + 1) F[j] |= nq;
    }
    // forced updates: a non-local (global) qubit some remaining gate needs
    // local at the next stage leaves the non-local (global) set
    double lb = popc(g & F[k]), lbg = popc(b & F[k]);
    for (int j = k + 1; j <= s - 2; j++) {
      lb += std::max(0, G - (n - popc(F[j])));
      lbg += std::max(0, Gg - (n - popc(F[j])));
    }
    return R == 0 ? unit * lb : lb + c * lbg;
  };
  for (int s = 2; s <= s_max && sfound < 0; s++) {
    const int lb0 = S.levels(empty, fwd, bwd);
    if (lb0 > s) continue;
    std::unordered_map<MemoKey, double, MemoHash> memo;
    std::vector<u64> pref, bpref;
    bool stop = false;
    double root_lb = 1e300;
    // node: stage k executed with non-local set g (global subset b),
    // frontier f, cost so far
    std::function<void(int, const Frontier &, u64, u64, double)> dfs = [&](int k, const Frontier &f, u64 g,
                                                                          u64 b, double cost) {
      if (stop) return;
      if (k == s - 2) {
        const u64 gl = final_global(g, all & ~S.remaining_nonins(f), G);
        if (gl == ~0ull) return;
        // the last global subset: keep what can stay, then the lowest
        u64 bl = b & gl;
        for (u64 p = gl & ~bl; p && popc(bl) < Gg; p &= p - 1) bl |= p & (~p + 1);
        const double tot = cost + step_cost(g, b, gl, bl);
        if (tot < best_cost) {
          best_cost = tot;
          best_pref = pref;
          best_pref.push_back(gl);
          best_bpref = bpref;
          best_bpref.push_back(bl);
          if (S.dbg) fprintf(stderr, "  s=%d plan cost %g evals %ld\n", s, tot, S.evals);
          if (best_cost <= root_lb) stop = true;
        }
        return;
      }
      const u64 cons = S.remaining_nonins(f);
      const u64 freeq = all & ~cons;
      const int kmin = std::max(0, G - popc(freeq));
      std::vector<u64> cand;
      for (int kk = kmin; kk <= std::min(G, popc(cons)); kk++) {
        combos(cons, kk, cons_sets);
        for (u64 cc : cons_sets) {
          const u64 g2 = fill_free(cc, k < 0 ? 0 : g, freeq, G, k < 0 ? 0 : b);
          if (g2 == ~0ull) continue;
          // more constrained globals than needed: when every newly global
          // one could be replaced by an unused free previous global (no
          // swap) the replacement is strictly cheaper and executes a superset
          const int newc = popc(cc & ~g);
          if (kk > kmin && k >= 0 && newc > 0 && newc <= popc(g & freeq & ~g2)) continue;
          cand.push_back(g2);
        }
      }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      std::vector<int> fw, bw;
      std::vector<u64> bsets;
      for (u64 g2 : cand) {
        if (stop) return;
        if (S.evals > S.budget) { S.over = true; stop = true; return; }
        Frontier f2 = f;
        if (S.maxexec(f2, all & ~g2) == 0) continue;
        const int need = S.levels(f2, fw, bw);
        if (need > s - 1 - (k + 1)) continue;
        global_subsets(g2, bsets);
        for (u64 b2 : bsets) {
          const double c2 = k < 0 ? 0.0 : cost + step_cost(g, b, g2, b2);
          if (c2 + lower_cost(s, k + 1, g2, b2, fw, bw) >= best_cost) continue;
          MemoKey key{f2, g2, b2, k + 1};
          auto it = memo.find(key);
          if (it != memo.end() && it->second <= c2) continue;
          memo[key] = c2;
          pref.push_back(g2);
          bpref.push_back(b2);
          dfs(k + 1, f2, g2, b2, c2);
          pref.pop_back();
          bpref.pop_back();
          if (stop) return;
        }
      }
    };
    // the cost bound at the root: every boundary's unavoidable swaps
    {
      std::vector<int> fw0, bw0;
      S.levels(empty, fw0, bw0);
      double lb = 0, lbg = 0;
      for (int j = 0; j <= s - 2; j++) {
        u64 Fj = 0;
        for (int x = 0; x < m; x++) {
          const int e = fw0[x], lat = s - 1 - bw0[x];
          if (e >= j && lat <= j + 1) Fj |= info[x].nonins;
        }
        lb += std::max(0, G - (n - popc(Fj)));
        lbg += std::max(0, Gg - (n - popc(Fj)));
      }
      root_lb = R == 0 ? unit * lb : lb + c * lbg;
    }
    dfs(-1, empty, 0, 0, 0.0);
    if (!best_pref.empty()) sfound = s;
    if (S.over) exact = false;
    if (S.dbg) fprintf(stderr, "s=%d found=%d cost %g root_lb %g evals %ld over %d\n", s, sfound, best_cost, root_lb, S.evals, (int)S.over);
    if (S.over && sfound < 0) {
      // budget exhausted without a plan at this s: look further (not exact)
      S.over = false;
      S.evals = 0;
    }
  }
  if (sfound < 0) fail(ATLAS_E_INFEASIBLE, "no staging with at most %d stages", s_max);
  const int sstar = sfound;
  sp.s = sstar;
  sp.cost = best_cost;
  sp.exact = exact;
  sp.global = best_bpref;
  for (u64 g : best_pref) sp.local.push_back(all & ~g);
  // replay maximal execution to assign gate stages
  Frontier f = empty;
  sp.gate_stage.assign(m, -1);
  for (int k = 0; k < sstar; k++) {
    Frontier before = f;
    S.maxexec(f, sp.local[k]);
    for (int g = 0; g < m; g++)
      if (S.done(f, g) && !S.done(before, g)) sp.gate_stage[g] = k;
  }
  for (int g = 0; g < m; g++)
    if (sp.gate_stage[g] < 0) fail(ATLAS_E_INFEASIBLE, "internal: staging replay incomplete");
  sp.states_explored = S.evals;
  return sp;
}

// The staging heuristic of SnuQS as PAPER.md describes it for its staging
// comparison ("greedily selects the qubits with more gates
// operating on non-local gates to form a stage and uses the number of total
// gates as a tiebreaker").  Reading (R32): every stage takes as
// local the L qubits with the most remaining gates that need them local
// (the qubit is a non-insular operand), ties broken by the number of
// remaining gates on the qubit, then by the lower index -- always including
// the non-insular qubits of the earliest pending gate, so that every stage
// makes progress; gates then run by maximal execution; repeat until every
// gate has run.  The baseline of the
// E5 experiment (tools/planner_experiments.py); option stager = 1.
StagePlan stage_greedy(int n, int L, int G, const std::vector<GateInfo> &info, int s_max, double c) {
  const int m = (int)info.size();
  for (int g = 0; g < m; g++)
    if (popc(info[g].nonins) > L)
      fail(ATLAS_E_INFEASIBLE, "gate %d has %d non-insular qubits > L = %d", g, popc(info[g].nonins), L);
  Search S;
  S.n = n; S.L = L; S.G = G; S.m = m; S.words = (m + 63) / 64; S.all = full_mask(n);
  S.info = &info; S.budget = 1;
  S.preds.resize(m);
  S.succs.resize(m);
  {
    std::vector<int> last(n, -1);
    for (int g = 0; g < m; g++)
      for (u64 q = info[g].qmask; q; q &= q - 1) {
        const int b = ctz(q);
        if (last[b] >= 0 && std::find(S.preds[g].begin(), S.preds[g].end(), last[b]) == S.preds[g].end())
          S.preds[g].push_back(last[b]);
        last[b] = g;
      }
  }
  StagePlan sp;
  Frontier f(S.words, 0);
  sp.gate_stage.assign(m, -1);
  u64 prevg = 0;
  int ndone = 0;
  for (int k = 0; ndone < m; k++) {
    if (k >= s_max) fail(ATLAS_E_INFEASIBLE, "greedy staging needs more than %d stages", s_max);
    std::vector<std::pair<std::pair<int, int>, int>> score;  // ((non-insular uses, uses), -q)
    std::vector<int> nonl(n, 0), uses(n, 0);
    for (int g = 0; g < m; g++) {
      if (S.done(f, g)) continue;
      for (u64 q = info[g].nonins; q; q &= q - 1) nonl[ctz(q)]++;
      for (u64 q = info[g].qmask; q; q &= q - 1) uses[ctz(q)]++;
    }
    std::vector<int> order(n);
    for (int q = 0; q < n; q++) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      if (nonl[a] != nonl[b]) return nonl[a] > nonl[b];
      if (uses[a] != uses[b]) return uses[a] > uses[b];
      return a < b;
    });
    // the non-insular qubits of the earliest pending gate are always local
    // (otherwise the ranking can stall on gates blocked behind it)
    u64 loc = 0;
    for (int g = 0; g < m; g++)
      if (!S.done(f, g)) {
        loc = info[g].nonins;
        break;
      }
    for (int i = 0; i < n && popc(loc) < L; i++) loc |= 1ull << order[i];
    const Frontier before = f;
    const int added = S.maxexec(f, loc);
    if (added == 0) fail(ATLAS_E_INFEASIBLE, "greedy staging made no progress at stage %d", k);
    for (int g = 0; g < m; g++)
      if (S.done(f, g) && !S.done(before, g)) sp.gate_stage[g] = k;
    ndone += added;
    const u64 gl = S.all & ~loc;
    sp.local.push_back(loc);
    sp.global.push_back(gl);
    if (k > 0) sp.cost += (1.0 + c) * popc(gl & ~prevg);
    prevg = gl;
  }
  sp.s = (int)sp.local.size();
  sp.exact = false;
  sp.states_explored = S.evals;
  return sp;
}

}  // namespace atlas
