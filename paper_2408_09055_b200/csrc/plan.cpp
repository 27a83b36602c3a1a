// plan.cpp -- Partition (Alg. 1) and lowering.
//
//   classify  -> stage (staging.cpp) -> placement + remap schedule
//   -> per stage: insular specialisation per rank -> Kernelize -> lowering to
//      device launches (fused matrices / shared-memory op programs).
//
// Placement (R6): stage 0 puts the local qubits that leave at the
// first remap in the top local slots; every remap swaps the top g' local slots
// with the incoming qubits' global slots (one all-to-all of contiguous blocks),
// preceded by a local bit-permutation ("pack") only when the outgoing qubits
// are not already in the top slots.
//
// Insular specialisation: a gate's global operands are insular
// (staging guarantees it) and their values are known per rank, so the gate
// restricted to those values is a smaller gate on its local operands, the
// identity, or a scalar.  An anti-diagonal gate on a global qubit is a
// relabelling: it toggles the qubit's flip bit (R14); the factor of
// Y-like gates becomes a per-rank scalar (R15).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstring>
#include <exception>
#include <map>
#include <sstream>
#include <tuple>

#include "ctx.h"

namespace atlas {

extern const char *kBuiltinModelC128;
extern const char *kBuiltinModelC64;
int shm_register_bits(int K);

CostModel builtin_cost_model(atlas_dtype dt) {
  return load_cost_model(dt == ATLAS_C128 ? kBuiltinModelC128 : kBuiltinModelC64, true);
}

namespace {

struct LGate {
  int nl = 0;
  int lq[3];        // local operands (logical), operand order
  Role lrole[3];
  cd M[64];         // 2^nl x 2^nl
  bool identity = false;
};

bool is_identity(const cd *M, int d) {
  for (int r = 0; r < d; r++)
    for (int c = 0; c < d; c++)
      if (std::abs(M[r * d + c] - (r == c ? cd(1) : cd(0))) > 1e-15) return false;
  return true;
}

// value of logical qubit q on rank `rank` during a stage (q global)
int global_value(const StageMap &mp, int L, int rank, int q, const std::vector<int> &flip) {
  int slot = mp.sigma[q];
  return ((rank >> (slot - L)) & 1) ^ flip[q];
}

enum PreKind { PK_DIAG = 0, PK_AFF = 1, PK_DENSE = 2 };

// one lowered block of a gate inside a shared-memory kernel
struct Pre {
  int type = OP_PHASE;
  int nt = 0;
  int ttile[2] = {0, 0};
  std::vector<std::pair<int, int>> sel;  // (physical slot, required value)
  std::vector<double> coef;
  bool swap = false;  // OP_DENSE2 that is the SWAP permutation
  int pk = PK_DENSE;
  u32 tsel = 0;       // tile bits of the selectors
  u32 tmask = 0;      // tile bits of the targets
  // a diagonal op conjugated through the phase's folded permutations:
  // c^(sum_k e_k * prod_{b in m_k} j_b) over monomials (m_k, e_k) of the
  // register-phase tile index j (|m_k| <= 2), times the base selectors
  bool conj = false;
  struct Mono {
    u32 m;       // tile bits of the monomial
    int e;       // exponent of c
    u64 bm, bv;  // tile-base condition under which it applies (0, 0: always)
  };
  std::vector<Mono> mono;
};

// A register phase under construction.  items: (0, dense ops) or
// (1, diagonal run), in execution order.  The affine map of the folded
// permutation gates: tile index j -> A j ^ c(base), A given by its columns.
struct PhaseB {
  u32 R = 0;
  std::vector<std::pair<int, std::vector<int>>> items;
  bool diag_open = false;
  u32 diag_bits = 0;
  bool has_perm = false;
  u32 PT = 0, PC = 0;  // tile bits targeted / used as controls by the folded gates
  u32 col[16];
  u32 c0 = 0;
  std::vector<std::tuple<u64, u64, u32>> terms;  // (base_mask, base_val, vector)
  PhaseB() {
    for (int b = 0; b < 16; b++) col[b] = 1u << b;
  }
  // Express a diagonal op that follows the folded permutations in the tile
  // index j the registers hold (D pi = pi D', D' = pi^-1 D pi): each tile
  // selector (x_a == v) becomes (parity(j & row_a(A)) ^ c0_a == v).
  // Supported: one selector with |row| <= 2, or two with |row| = 1.
  //
  // Base-conditioned folded gates (a CX whose control is a non-active qubit:
  // term (single base bit, value) with vector e_a) flip selector a per tile;
  // every combination of those base bits (<= 4) gets its own monomials under
  // that base condition.
  bool conjugate(const Pre &p, const std::vector<int> &tile_of_slot, int K, Pre &out) const {
    struct Sel {
      u32 row;
      int w;      // required parity with all flip bits 0
      u64 flips;  // base bits whose value XORs into the parity
    };
    std::vector<Sel> sels;
    u64 U = 0;
    for (auto &sv : p.sel) {
      int a = tile_of_slot[sv.first];
      if (a < 0) continue;
      Sel s{0, sv.second ^ (int)((c0 >> a) & 1), 0};
      for (auto &t : terms)
        if ((std::get<2>(t) >> a) & 1) {
          const u64 bm = std::get<0>(t), bv = std::get<1>(t);
          if (popc(bm) != 1) return false;
          // [base & bm == bv] = base_bit ^ (bv == 0)
          s.flips ^= bm;
          if (bv == 0) s.w ^= 1;
        }
      for (int b = 0; b < K; b++)
        if ((col[b] >> a) & 1) s.row |= 1u << b;
      U |= s.flips;
      sels.push_back(s);
    }
    if (popc(U) > 4) return false;
    bool shape_ok = (sels.size() == 1 && popc((u64)sels[0].row) <= 2) ||
                    (sels.size() == 2 && popc((u64)sels[0].row) == 1 &&
                     popc((u64)sels[1].row) == 1 && sels[0].row != sels[1].row);
    if (!shape_ok) return false;
    out = p;
    out.conj = true;
    out.mono.clear();
    std::vector<int> ub;
    for (int b = 0; b < 64; b++)
      if ((U >> b) & 1) ub.push_back(b);
    for (int z = 0; z < (1 << ub.size()); z++) {
      u64 bv = 0;
      for (size_t i = 0; i < ub.size(); i++)
        if ((z >> i) & 1) bv |= 1ull << ub[i];
      auto wv = [&](const Sel &s) { return s.w ^ (popc(s.flips & bv) & 1); };
      std::vector<std::pair<u32, int>> mm;
      if (sels.size() == 1) {
        u32 r = sels[0].row;
        int w = wv(sels[0]);
        if (popc((u64)r) == 1) {
          if (w) mm = {{r, 1}};
          else mm = {{0u, 1}, {r, -1}};
        } else {
          u32 a = r & (~r + 1), b = r ^ a;
          if (w) mm = {{a, 1}, {b, 1}, {r, -2}};
          else mm = {{0u, 1}, {a, -1}, {b, -1}, {r, 2}};
        }
      } else {
        u32 a = sels[0].row, b = sels[1].row;
        int va = wv(sels[0]), vb = wv(sels[1]);
        // [j_a == va][j_b == vb] expanded
        if (va && vb) mm = {{a | b, 1}};
        else if (va && !vb) mm = {{a, 1}, {a | b, -1}};
        else if (!va && vb) mm = {{b, 1}, {a | b, -1}};
        else mm = {{0u, 1}, {a, -1}, {b, -1}, {a | b, 1}};
      }
      for (auto &x : mm) out.mono.push_back(Pre::Mono{x.first, x.second, U, bv});
    }
    out.tsel = 0;
    for (auto &m : out.mono) out.tsel |= m.m;
    return true;
  }
  // tile bits the net folded map moves or reads: a later op may run before
  // the map only if its bits avoid these
  u32 touched(int K) const {
    u32 t = c0;
    for (auto &tm : terms) t |= std::get<2>(tm);
    for (int b = 0; b < K; b++)
      if (col[b] != (1u << b)) t |= col[b] | (1u << b);
    return t;
  }
  bool aff_identity(int K) const {
    for (int b = 0; b < K; b++)
      if (col[b] != (1u << b)) return false;
    return c0 == 0 && terms.empty();
  }
  // compose x -> x ^ [x_c == v] e_t (CX), x -> x ^ e_t (X, optionally
  // conditioned on tile-base bits), or the swap of tile bits a and b
  void aff_apply(const Pre &p, const std::vector<int> &tile_of_slot, int K) {
    has_perm = true;
    auto lin_cx = [&](u32 x, int c, int t) { return ((x >> c) & 1) ? (x ^ (1u << t)) : x; };
    auto lin_swap = [&](u32 x, int a, int b) {
      u32 xa = (x >> a) & 1, xb = (x >> b) & 1;
      if (xa != xb) x ^= (1u << a) | (1u << b);
      return x;
    };
    if (p.type == OP_DENSE2) {  // SWAP
      const int a = p.ttile[0], b = p.ttile[1];
      for (int i = 0; i < K; i++) col[i] = lin_swap(col[i], a, b);
      c0 = lin_swap(c0, a, b);
      for (auto &t : terms) std::get<2>(t) = lin_swap(std::get<2>(t), a, b);
      PT |= (1u << a) | (1u << b);
      return;
    }
    const int t = p.ttile[0];
    PT |= 1u << t;
    int ctile = -1, cval = 1;
    u64 bm = 0, bv = 0;
    for (auto &sv : p.sel) {
      int tb = tile_of_slot[sv.first];
      if (tb >= 0) {
        ctile = tb;
        cval = sv.second;
      } else {
        bm |= 1ull << sv.first;
        bv |= (u64)sv.second << sv.first;
      }
    }
    if (ctile >= 0) {
      PC |= 1u << ctile;
      for (int i = 0; i < K; i++) col[i] = lin_cx(col[i], ctile, t);
      c0 = lin_cx(c0, ctile, t);
      if (!cval) c0 ^= 1u << t;
      for (auto &tm : terms) std::get<2>(tm) = lin_cx(std::get<2>(tm), ctile, t);
    } else if (bm == 0) {
      c0 ^= 1u << t;
    } else {
      terms.push_back(std::make_tuple(bm, bv, 1u << t));
    }
  }
};

u64 ls_logical(const std::vector<int> &sigma, int ls) {
  u64 s = 0;
  for (int q = 0; q < (int)sigma.size(); q++)
    if (sigma[q] < ls) s |= 1ull << q;
  return s;
}

}  // namespace

void build_plan(atlas_ctx *C, int s_max, double cf) {
  auto t0 = std::chrono::steady_clock::now();
  const int n = C->n, L = C->L, G = C->G, m = (int)C->gates.size();
  // ---- cost model
  C->cm = C->opt.cost_model.empty() ? builtin_cost_model(C->dt)
                                    : load_cost_model(C->opt.cost_model, false);
  if (C->opt.shm_qubits >= 0) C->cm.q_max_shared = C->opt.shm_qubits;
  if (C->opt.fusion_qubits >= 0) C->cm.q_max_fusion = C->opt.fusion_qubits;
  if (C->opt.ls_qubits >= 0) C->cm.ls_qubits = C->opt.ls_qubits;
  C->cm.q_max_fusion = std::min(C->cm.q_max_fusion, 5);   // fused templates k <= 5
  C->cm.q_max_shared = std::min(C->cm.q_max_shared, 13);  // shm templates K <= 13
  if ((int)C->cm.fusion_cost.size() < C->cm.q_max_fusion)
    fail(ATLAS_E_INVALID, "cost model fusion table too short");
  // ---- a1: insular classification
  C->info.resize(m);
  for (int g = 0; g < m; g++) C->info[g] = classify(C->gates[g]);
  // ---- a2: staging
  C->c = cf;
  // the staging depends only on the circuit, L, G, s_max, c and the budget:
  // reuse it when atlas_plan rebuilds the plan for another ls_qubits (ls_auto)
  if (C->sp_key_valid && C->sp_key_smax == s_max && C->sp_key_c == cf &&
      C->sp_key_budget == C->opt.stage_budget && C->sp_key_stager == C->opt.stager &&
      C->sp_key_regional == C->opt.regional) {
    // stage_us keeps the time of the staging that is reused
  } else {
    C->sp = C->opt.stager == 1 ? stage_greedy(n, L, G, C->info, s_max, cf)
                               : stage_circuit(n, L, G, C->info, s_max, cf, C->opt.stage_budget,
                                               C->opt.regional);
    C->stage_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    C->sp_key_valid = true;
    C->sp_key_smax = s_max;
    C->sp_key_c = cf;
    C->sp_key_budget = C->opt.stage_budget;
    C->sp_key_stager = C->opt.stager;
    C->sp_key_regional = C->opt.regional;
  }
  const int s = C->sp.s;
  C->stage_gates.assign(s, {});
  for (int g = 0; g < m; g++) C->stage_gates[C->sp.gate_stage[g]].push_back(g);
  // ---- placement and remap schedule
  C->maps.assign(s, {});
  C->exch.assign(s, {});
  {
    std::vector<int> sigma(n, -1), flip(n, 0);
    u64 loc0 = C->sp.local[0];
    u64 out1 = s > 1 ? (loc0 & ~C->sp.local[1]) : 0;
    int slot = 0;
    for (int q = 0; q < n; q++)
      if (((loc0 >> q) & 1) && !((out1 >> q) & 1)) sigma[q] = slot++;
    for (int q = 0; q < n; q++)
      if ((out1 >> q) & 1) sigma[q] = slot++;
    for (int q = 0; q < n; q++)
      if (!((loc0 >> q) & 1)) sigma[q] = slot++;
    C->maps[0].sigma = sigma;
    C->maps[0].flip_begin = flip;
  }
  // flips evolve inside a stage (anti-diagonal gates on global qubits); the
  // end-of-stage flips are filled by the specialisation pass below, and the
  // next stage's mapping is derived from them, so do both per stage.
  C->K_tile = 0;
  {
    int qms = std::min(C->cm.q_max_shared, L);
    C->K_tile = (qms >= 6 && (C->opt.kinds & 2)) ? qms : 0;
  }
  C->nslots = (C->opt.virtual_world && C->world > 1) ? C->world : 1;
  C->prog.assign(C->nslots, {});
  C->coef.clear();
  C->ops.clear();
  C->phases.clear();
  C->mats.clear();
  C->newpos.clear();
  C->kplans.assign(s, {});
  const int B = C->dt == ATLAS_C128 ? 16 : 8;
  const int64_t pass_bytes = 2 * ((int64_t)B << L);
  auto slot_rank = [&](int sl) { return C->nslots > 1 ? sl : C->rank; };

  // Three passes over the stages: (A) placement, remap launches and the
  // insular specialisation (the next stage's mapping depends on the flips
  // this produces, not on kernelization), (B) Kernelize of every stage on
  // host threads (independent; each deterministic), (C) lowering.
  struct StageWork {
    std::vector<std::vector<Launch>> pre;   // pack / exchange launches per slot
    std::vector<std::vector<LGate>> lg;
    std::vector<cd> scalar;
    std::vector<KGate> seq;
    std::vector<int> seq_pos;
    KernelizeOptions ko;
    KernelPlan kp;
  };
  std::vector<StageWork> SW(s);
  for (int k = 0; k < s; k++) {
    StageMap &mp = C->maps[k];
    SW[k].pre.assign(C->nslots, {});
    // ---- remap from stage k-1
    if (k > 0) {
      const StageMap &pm = C->maps[k - 1];
      std::vector<int> sigma = pm.sigma, flip = pm.flip_end;
      u64 O = C->sp.local[k - 1] & ~C->sp.local[k];
      u64 I = C->sp.local[k] & ~C->sp.local[k - 1];
      int gp = popc(O);
      Exchange &ex = C->exch[k];
      ex.gp = gp;
      // pack if the outgoing qubits are not exactly the top gp local slots
      std::vector<int> at(n, -1);
      for (int q = 0; q < n; q++) at[sigma[q]] = q;
      bool ok = true;
      for (int j = 0; j < gp; j++)
        if (!((O >> at[L - gp + j]) & 1)) ok = false;
      if (!ok && gp > 0) {
        std::vector<int> newslot(n);
        for (int i = 0; i < n; i++) newslot[i] = i;
        std::vector<int> vac, disp;
        std::vector<int> outs;
        for (int q = 0; q < n; q++)
          if ((O >> q) & 1) outs.push_back(q);
        for (int q : outs)
          if (sigma[q] < L - gp) vac.push_back(sigma[q]);
        for (int sl = L - gp; sl < L; sl++)
          if (!((O >> at[sl]) & 1)) disp.push_back(sl);
        std::sort(vac.begin(), vac.end());
        std::sort(disp.begin(), disp.end());
        for (size_t i = 0; i < disp.size(); i++) newslot[disp[i]] = vac[i];
        // outgoing qubits fill the top slots in ascending logical order
        int j = 0;
        for (int q : outs) newslot[sigma[q]] = L - gp + (j++);
        // check it is a permutation of the local slots
        std::vector<int> seen(L, 0);
        for (int i = 0; i < L; i++) seen[newslot[i]]++;
        for (int i = 0; i < L; i++)
          if (seen[i] != 1) fail(ATLAS_E_INVALID, "internal: pack is not a permutation");
        int64_t off = (int64_t)C->newpos.size();
        for (int i = 0; i < L; i++) C->newpos.push_back(newslot[i]);
        for (int q = 0; q < n; q++) sigma[q] = newslot[sigma[q]];
        for (int sl = 0; sl < C->nslots; sl++) {
          Launch ln;
          ln.type = L_PACK;
          ln.stage = k;
          ln.newpos_off = off;
          ln.bytes = pass_bytes;
          SW[k].pre[sl].push_back(ln);
        }
        ex.packed = true;
        for (int q = 0; q < n; q++) at[sigma[q]] = q;
      }
      std::vector<int> ins;
      for (int q = 0; q < n; q++)
        if ((I >> q) & 1) ins.push_back(q);
      ex.gamma.clear();
      ex.fI.clear();
      for (int j = 0; j < gp; j++) {
        int oq = at[L - gp + j], iq = ins[j];
        int gslot = sigma[iq];
        ex.gamma.push_back(gslot - L);
        ex.fI.push_back(flip[iq]);
        sigma[iq] = L - gp + j;
        sigma[oq] = gslot;
        flip[iq] = 0;
        flip[oq] = 0;
      }
      if (gp > 0)
        for (int sl = 0; sl < C->nslots; sl++) {
          Launch ln;
          ln.type = L_EXCHANGE;
          ln.stage = k;
          ln.bytes = (int64_t)(((double)(B) * (double)(1ull << L)) * (1.0 - std::ldexp(1.0, -gp)));
          SW[k].pre[sl].push_back(ln);
        }
      mp.sigma = sigma;
      mp.flip_begin = flip;
    }
    // ---- insular specialisation, in circuit order, per simulated rank
    const std::vector<int> &ids = C->stage_gates[k];
    std::vector<int> flip = mp.flip_begin;
    std::vector<std::vector<LGate>> &lg = SW[k].lg;
    lg.assign(C->nslots, std::vector<LGate>(ids.size()));
    std::vector<cd> &scalar = SW[k].scalar;
    scalar.assign(C->nslots, cd(1));
    std::vector<KGate> &seq = SW[k].seq;
    std::vector<int> &seq_pos = SW[k].seq_pos;  // position in ids
    for (size_t ii = 0; ii < ids.size(); ii++) {
      const Gate &g = C->gates[ids[ii]];
      const GateInfo &gi = C->info[ids[ii]];
      const int ka = kind_arity(g.kind);
      cd M[64];
      gate_matrix(g, M);
      const int d = 1 << ka;
      int nl = 0;
      for (int j = 0; j < ka; j++)
        if (mp.sigma[g.q[j]] < L) nl++;
      if (nl == 0) {
        // every operand global and insular
        if (ka == 1 && gi.role[0] == ANTI) {
          int q = g.q[0];
          for (int sl = 0; sl < C->nslots; sl++) {
            int v_new = global_value(mp, L, slot_rank(sl), q, flip) ^ 1;
            scalar[sl] *= M[v_new * 2 + (1 - v_new)];
          }
          flip[q] ^= 1;
        } else {
          for (int sl = 0; sl < C->nslots; sl++) {
            int sel = 0;
            for (int j = 0; j < ka; j++)
              sel |= global_value(mp, L, slot_rank(sl), g.q[j], flip) << j;
            scalar[sl] *= M[sel * d + sel];
          }
        }
        continue;
      }
      KGate kg;
      kg.gid = ids[ii];
      kg.qubits = kg.active = kg.diagq = kg.antiq = 0;
      kg.kind = g.kind;
      for (int j = 0; j < ka; j++) {
        int q = g.q[j];
        if (mp.sigma[q] >= L) {
          if (gi.role[j] == TGT || gi.role[j] == ANTI)
            fail(ATLAS_E_INVALID, "internal: non-insular operand of gate %d is global", ids[ii]);
          continue;
        }
        kg.qubits |= 1ull << q;
        if (gi.role[j] == TGT || gi.role[j] == ANTI) kg.active |= 1ull << q;
        if (gi.role[j] == ANTI) kg.antiq |= 1ull << q;
        if (gi.role[j] == CTL || gi.role[j] == DIAG) kg.diagq |= 1ull << q;
      }
      seq.push_back(kg);
      seq_pos.push_back((int)ii);
      for (int sl = 0; sl < C->nslots; sl++) {
        LGate &x = lg[sl][ii];
        x.nl = 0;
        int kv[3], lpos[3];
        for (int j = 0; j < ka; j++) {
          int q = g.q[j];
          if (mp.sigma[q] >= L) {
            kv[j] = global_value(mp, L, slot_rank(sl), q, flip);
            lpos[j] = -1;
          } else {
            kv[j] = -1;
            lpos[j] = x.nl;
            x.lq[x.nl] = q;
            x.lrole[x.nl] = gi.role[j];
            x.nl++;
          }
        }
        const int dl = 1 << x.nl;
        for (int r = 0; r < dl; r++)
          for (int c = 0; c < dl; c++) {
            int R = 0, Cc = 0;
            for (int j = 0; j < ka; j++) {
              int br = kv[j] >= 0 ? kv[j] : ((r >> lpos[j]) & 1);
              int bc = kv[j] >= 0 ? kv[j] : ((c >> lpos[j]) & 1);
              R |= br << j;
              Cc |= bc << j;
            }
            x.M[r * dl + c] = M[R * d + Cc];
          }
        x.identity = is_identity(x.M, dl);
      }
    }
    mp.flip_end = flip;
    // ---- a3: kernelization options of the stage
    KernelizeOptions &ko = SW[k].ko;
    ko.algo = C->opt.kernelizer;
    ko.prune_T = C->opt.prune_T;
    ko.lift = C->opt.lift != 0;
    ko.attach = C->opt.attach != 0;
    ko.kinds = C->opt.kinds;
    ko.front = C->opt.front != 0;
    ko.dp_budget = C->opt.dp_budget;
    ko.L = L;
    ko.ls_set = ls_logical(mp.sigma, std::min(C->cm.ls_qubits, L));
  }
  // ---- (B) a3: Kernelize every stage, stages spread over host threads
  {
    std::atomic<int> next{0};
    std::vector<std::exception_ptr> errs(s);
    auto worker = [&]() {
      for (;;) {
        const int k = next.fetch_add(1);
        if (k >= s) return;
        try {
          StageWork &w = SW[k];
          if (w.seq.empty()) continue;
          if (w.ko.algo == 1) w.kp = ordered_kernelize(w.seq, C->cm, w.ko);
          else if (w.ko.algo == 2) w.kp = greedy_kernelize(w.seq, C->cm, w.ko);
          else if (w.ko.algo == 3) w.kp = front_kernelize(w.seq, C->cm, w.ko);
          else if (w.ko.algo == 4) w.kp = dp_only_kernelize(w.seq, C->cm, w.ko);
          else w.kp = dp_kernelize(w.seq, C->cm, w.ko);
        } catch (...) {
          errs[k] = std::current_exception();
        }
      }
    };
    unsigned nth = std::thread::hardware_concurrency();
    nth = std::max(1u, std::min<unsigned>(nth ? nth : 1, (unsigned)s));
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nth; t++) th.emplace_back(worker);
    worker();
    for (auto &t : th) t.join();
    for (int k = 0; k < s; k++)
      if (errs[k]) std::rethrow_exception(errs[k]);
  }
  // ---- (C) lowering
  for (int k = 0; k < s; k++) {
    StageMap &mp = C->maps[k];
    for (int sl = 0; sl < C->nslots; sl++)
      for (auto &ln : SW[k].pre[sl]) C->prog[sl].push_back(ln);
    std::vector<std::vector<LGate>> &lg = SW[k].lg;
    std::vector<cd> &scalar = SW[k].scalar;
    std::vector<KGate> &seq = SW[k].seq;
    std::vector<int> &seq_pos = SW[k].seq_pos;
    const KernelPlan &kp = SW[k].kp;
    // kernel gate indices are positions in seq; keep them for lowering and
    // translate to circuit ids for the plan report
    C->kplans[k] = kp;
    for (auto &K : C->kplans[k].kernels)
      for (auto &gidx : K.gates) gidx = seq[gidx].gid;
    // ---- a4: lowering per simulated rank
    for (int sl = 0; sl < C->nslots; sl++) {
      bool scalar_done = std::abs(scalar[sl] - cd(1)) < 1e-15;
      for (const Kernel &K : kp.kernels) {
        // skip kernels that are the identity on this rank
        bool all_id = true;
        for (int gi : K.gates)
          if (!lg[sl][seq_pos[gi]].identity) all_id = false;
        if (all_id && scalar_done) continue;
        Launch ln;
        ln.stage = k;
        ln.bytes = pass_bytes;
        if (K.kind == K_FUSION) {
          ln.type = L_FUSED;
          std::vector<int> slots;
          u64 qs = K.qubits;
          while (qs) {
            int q = ctz(qs);
            qs &= qs - 1;
            slots.push_back(mp.sigma[q]);
          }
          std::sort(slots.begin(), slots.end());
          const int kk = (int)slots.size();
          const int D = 1 << kk;
          ln.fl.k = kk;
          for (int j = 0; j < 6; j++) ln.fl.t[j] = j < kk ? slots[j] : 0;
          // matrix = product of the member gates in kernel order
          std::vector<cd> U(D * D, cd(0));
          for (int i = 0; i < D; i++) U[i * D + i] = 1;
          for (int gi : K.gates) {
            const LGate &x = lg[sl][seq_pos[gi]];
            if (x.identity) continue;
            int bitpos[3];
            for (int j = 0; j < x.nl; j++)
              bitpos[j] = (int)(std::find(slots.begin(), slots.end(), mp.sigma[x.lq[j]]) - slots.begin());
            const int dl = 1 << x.nl;
            int mask = 0;
            for (int j = 0; j < x.nl; j++) mask |= 1 << bitpos[j];
            for (int col = 0; col < D; col++) {
              for (int b = 0; b < D; b++) {
                if (b & mask) continue;
                cd v[8], w[8];
                for (int c = 0; c < dl; c++) {
                  int idx = b;
                  for (int j = 0; j < x.nl; j++)
                    if ((c >> j) & 1) idx |= 1 << bitpos[j];
                  v[c] = U[idx * D + col];
                }
                for (int r = 0; r < dl; r++) {
                  w[r] = 0;
                  for (int c = 0; c < dl; c++) w[r] += x.M[r * dl + c] * v[c];
                }
                for (int r = 0; r < dl; r++) {
                  int idx = b;
                  for (int j = 0; j < x.nl; j++)
                    if ((r >> j) & 1) idx |= 1 << bitpos[j];
                  U[idx * D + col] = w[r];
                }
              }
            }
          }
          if (!scalar_done) {
            for (auto &z : U) z *= scalar[sl];
            scalar_done = true;
          }
          ln.fl.mat_off = (int64_t)C->mats.size();
          for (auto &z : U) C->mats.push_back(make_double2(z.real(), z.imag()));
        } else {
          ln.type = L_SHM;
          const int K_ = C->K_tile;
          const int RB = (K_ == 12 && C->opt.shm_rb == 3) ? 3 : shm_register_bits(K_);
          // active slots: kernel qubits (active set + LSB) padded to K_ slots
          u64 amask = 0;
          u64 qs = K.qubits;
          while (qs) {
            int q = ctz(qs);
            qs &= qs - 1;
            amask |= 1ull << mp.sigma[q];
          }
          for (int sl2 = 0; sl2 < L && popc(amask) < K_; sl2++) amask |= 1ull << sl2;
          if (popc(amask) != K_) fail(ATLAS_E_INVALID, "internal: shm active set %d != K %d", popc(amask), K_);
          std::vector<int> act;
          for (int b = 0; b < L; b++)
            if ((amask >> b) & 1) act.push_back(b);
          std::vector<int> tile_of_slot(L, -1);
          for (int b = 0; b < K_; b++) tile_of_slot[act[b]] = b;
          ln.sl = ShmLaunch{};
          ln.sl.out_perm_off = -1;
          ln.sl.K = K_;
          ln.sl.RB = RB;
          ln.sl.nbuf = (C->dt == ATLAS_C128 && K_ == 13) ? 1 : C->opt.shm_nbuf;
          for (int b = 0; b < 16; b++) ln.sl.act[b] = b < K_ ? act[b] : 0;
          const u64 lmask = (L == 64) ? ~0ull : ((1ull << L) - 1);
          ln.sl.nonactive = lmask & ~amask;
          ln.sl.ntiles = 1ull << (L - K_);
          // ---- ops before register assignment
          std::vector<Pre> pre;
          if (!scalar_done) {
            Pre p;
            p.type = OP_PHASE;
            p.coef = {scalar[sl].real(), scalar[sl].imag()};
            pre.push_back(p);
            scalar_done = true;
          }
          for (int gi : K.gates) {
            const LGate &x = lg[sl][seq_pos[gi]];
            if (x.identity) continue;
            int tj[3], sj[3], nt = 0, ns = 0;
            for (int j = 0; j < x.nl; j++) {
              if (x.lrole[j] == TGT || x.lrole[j] == ANTI) tj[nt++] = j;
              else sj[ns++] = j;
            }
            if (nt > 2) fail(ATLAS_E_UNSUPPORTED, "internal: gate with %d targets in shm kernel", nt);
            const int dl = 1 << x.nl;
            const int dt = 1 << nt;
            for (int sv = 0; sv < (1 << ns); sv++) {
              cd blk[16];
              bool ident = true;
              for (int r = 0; r < dt; r++)
                for (int c = 0; c < dt; c++) {
                  int R = 0, Cc = 0;
                  for (int a = 0; a < nt; a++) {
                    R |= ((r >> a) & 1) << tj[a];
                    Cc |= ((c >> a) & 1) << tj[a];
                  }
                  for (int a = 0; a < ns; a++) {
                    R |= ((sv >> a) & 1) << sj[a];
                    Cc |= ((sv >> a) & 1) << sj[a];
                  }
                  blk[r * dt + c] = x.M[R * dl + Cc];
                  if (std::abs(blk[r * dt + c] - (r == c ? cd(1) : cd(0))) > 1e-15) ident = false;
                }
              if (ident) continue;
              Pre p;
              p.nt = nt;
              for (int a = 0; a < ns; a++) p.sel.push_back({mp.sigma[x.lq[sj[a]]], (sv >> a) & 1});
              for (int a = 0; a < nt; a++) {
                int ts = tile_of_slot[mp.sigma[x.lq[tj[a]]]];
                if (ts < 0) fail(ATLAS_E_INVALID, "internal: shm target not active");
                p.ttile[a] = ts;
              }
              if (nt == 0) {
                p.type = OP_PHASE;
                p.coef = {blk[0].real(), blk[0].imag()};
              } else if (nt == 1) {
                bool isx = std::abs(blk[0]) < 1e-15 && std::abs(blk[3]) < 1e-15 &&
                           std::abs(blk[1] - cd(1)) < 1e-15 && std::abs(blk[2] - cd(1)) < 1e-15;
                p.type = isx ? OP_PERM1 : OP_DENSE1;
                if (!isx)
                  for (int i = 0; i < 4; i++) {
                    p.coef.push_back(blk[i].real());
                    p.coef.push_back(blk[i].imag());
                  }
                // A complex 2x2 unitary block = D1 R D2 with R real and D1,
                // D2 diagonal (Euler ZYZ form): the real block costs half the
                // flops of the complex one, and the diagonal factors join the
                // phase's diagonal runs (one multiply per element per run).
                bool split = false;
                cd d0, d1, e1;
                double r[4];
                if (!isx && C->opt.shm_split_dense) {
                  // worth it only when the complex block has more nonzero
                  // real/imaginary parts than the 4 of a real block (RX's
                  // entries are each real or imaginary: no gain)
                  bool tiny = false;
                  int parts = 0;
                  for (int i = 0; i < 4; i++) {
                    parts += (blk[i].real() != 0.0) + (blk[i].imag() != 0.0);
                    if (std::abs(blk[i]) < 1e-9) tiny = true;
                  }
                  if (parts > 4 && !tiny) {
                    r[0] = std::abs(blk[0]);
                    r[2] = std::abs(blk[2]);
                    d0 = blk[0] / r[0];
                    d1 = blk[2] / r[2];
                    r[1] = -std::abs(blk[1]);
                    e1 = blk[1] / d0 / r[1];
                    const cd r3 = blk[3] / (d1 * e1);
                    r[3] = r3.real();
                    double err = std::abs(r3.imag()) + std::abs(std::abs(e1) - 1.0);
                    const cd rec[4] = {d0 * r[0], d0 * r[1] * e1, d1 * r[2], d1 * r[3] * e1};
                    for (int i = 0; i < 4; i++) err += std::abs(rec[i] - blk[i]);
                    split = err < 1e-13;
                  }
                }
                if (split) {
                  const int ts = mp.sigma[x.lq[tj[0]]];
                  Pre pd2 = p, pd1a = p, pd1b = p;
                  pd2.type = pd1a.type = pd1b.type = OP_PHASE;
                  pd2.nt = pd1a.nt = pd1b.nt = 0;
                  pd2.sel.push_back({ts, 1});
                  pd2.coef = {e1.real(), e1.imag()};
                  pd1a.coef = {d0.real(), d0.imag()};
                  const cd q = d1 / d0;
                  pd1b.sel.push_back({ts, 1});
                  pd1b.coef = {q.real(), q.imag()};
                  if (std::abs(e1 - cd(1)) > 1e-15) pre.push_back(pd2);
                  p.coef.clear();
                  for (int i = 0; i < 4; i++) {
                    p.coef.push_back(r[i]);
                    p.coef.push_back(0.0);
                  }
                  pre.push_back(p);
                  if (std::abs(d0 - cd(1)) > 1e-15) pre.push_back(pd1a);
                  if (std::abs(q - cd(1)) > 1e-15) pre.push_back(pd1b);
                  continue;
                }
              } else {
                p.type = OP_DENSE2;
                if (p.ttile[0] > p.ttile[1]) {  // canonical order t0 < t1
                  std::swap(p.ttile[0], p.ttile[1]);
                  cd b2[16];
                  for (int r = 0; r < 4; r++)
                    for (int c = 0; c < 4; c++) {
                      int rs = ((r & 1) << 1) | (r >> 1), cs = ((c & 1) << 1) | (c >> 1);
                      b2[rs * 4 + cs] = blk[r * 4 + c];
                    }
                  std::copy(b2, b2 + 16, blk);
                }
                bool isswap = true;
                const int sw[4] = {0, 2, 1, 3};
                for (int r = 0; r < 4; r++)
                  for (int c = 0; c < 4; c++)
                    if (std::abs(blk[r * 4 + c] - (c == sw[r] ? cd(1) : cd(0))) > 1e-15) isswap = false;
                p.swap = isswap;
                for (int i = 0; i < 16; i++) {
                  p.coef.push_back(blk[i].real());
                  p.coef.push_back(blk[i].imag());
                }
              }
              pre.push_back(p);
            }
          }
          // ---- classify: diagonal / affine permutation (folded into the
          // phase's store addresses) / dense (needs register residency)
          for (Pre &p : pre) {
            u32 tsel = 0;
            int nts = 0, nbs = 0;
            for (auto &sv : p.sel) {
              int tb = tile_of_slot[sv.first];
              if (tb >= 0) {
                tsel |= 1u << tb;
                nts++;
              } else {
                nbs++;
              }
            }
            p.tsel = tsel;
            if (p.type == OP_PHASE) p.pk = PK_DIAG;
            else if (p.type == OP_PERM1 && (nts == 0 || (nts == 1 && nbs == 0))) p.pk = PK_AFF;
            else if (p.type == OP_DENSE2 && p.swap && p.sel.empty()) p.pk = PK_AFF;
            else p.pk = PK_DENSE;
            p.tmask = 0;
            for (int a = 0; a < p.nt; a++) p.tmask |= 1u << p.ttile[a];
          }
          // ---- register phases: dense ops need their target
          // tile bits in registers (<= RB per phase); diagonal runs become
          // factor slots; affine permutations are composed into the phase's
          // store map.  Ops are only reordered across ops they commute with.
          std::vector<PhaseB> phs(1);
          const int npre = (int)pre.size();
          // a diagonal op whose tile selectors are not register bits of the
          // current phase waits for the next dense op: if that op starts a
          // new phase the diagonal op opens it (its selectors are then
          // register bits there, and it joins the literal per-element factors
          // instead of a per-thread runtime factor on every element); else it
          // is placed in the current phase as before.  Program order is kept:
          // it runs after every op of the current phase.
          std::vector<int> pend;
          PhaseB *cur = &phs.back();
          auto fresh = [&]() {
            phs.emplace_back();
            cur = &phs.back();
          };
          auto place_diag = [&](int i) {
            const Pre &p = pre[i];
            int idx = i;
            if (cur->has_perm && (p.tsel & cur->touched(K_))) {
              Pre q;
              if (cur->conjugate(p, tile_of_slot, K_, q)) {
                pre.push_back(q);
                idx = (int)pre.size() - 1;
              } else {
                fresh();
              }
            }
            // hoist into the earliest diagonal run it can reach: it
            // commutes with every dense op whose targets avoid its bits
            // (all ops of a phase act on the pre-map tile index)
            const u32 bits = pre[idx].tsel;
            int cand = -1;
            int at = (int)cur->items.size();
            if (C->opt.shm_hoist_diag) {
              for (int k2 = (int)cur->items.size() - 1; k2 >= 0; k2--) {
                auto &it = cur->items[k2];
                if (it.first == 1) {
                  cand = k2;
                  continue;
                }
                bool blocks = false;
                for (int o2 : it.second)
                  if (pre[o2].tmask & bits) blocks = true;
                if (blocks) break;
                at = k2;
              }
            }
            const int last = (int)cur->items.size() - 1;
            if (cand >= 0 && (cand != last || cur->diag_open)) {
              cur->items[cand].second.push_back(idx);
              if (cand == last) cur->diag_bits |= bits;
              return;
            }
            if (!C->opt.shm_hoist_diag || at >= (int)cur->items.size()) {
              if (!cur->diag_open) {
                cur->items.push_back({1, {}});
                cur->diag_open = true;
                cur->diag_bits = 0;
              }
              cur->items.back().second.push_back(idx);
              cur->diag_bits |= bits;
            } else {
              cur->items.insert(cur->items.begin() + at, {1, {idx}});
            }
          };
          auto flush = [&]() {
            for (int j : pend) place_diag(j);
            pend.clear();
          };
          for (int i = 0; i < npre; i++) {
            const Pre p = pre[i];
            bool explicit_perm = false;
            if (p.pk == PK_AFF && p.type == OP_PERM1 && C->opt.shm_explicit_perm &&
                popc((u64)(cur->R | p.tmask)) <= RB) {
              // Folding it would make a later dense op on its bits start a
              // new phase; when such an op comes before the phase fills up,
              // swap the registers explicitly instead (a few moves).
              u32 rs = cur->R | p.tmask;
              for (int q = i + 1; q < npre; q++) {
                const Pre &pq = pre[q];
                if (pq.pk != PK_DENSE) continue;
                if (pq.tmask & (p.tmask | p.tsel)) {
                  explicit_perm = true;
                  break;
                }
                rs |= pq.tmask;
                if (popc((u64)rs) > RB) break;
              }
            }
            if (p.pk == PK_AFF && !explicit_perm) {
              flush();
              cur->aff_apply(p, tile_of_slot, K_);
              if (cur->aff_identity(K_)) cur->has_perm = false;  // e.g. CX RZ CX
              continue;
            }
            if (p.pk == PK_DIAG) {
              if (C->opt.shm_defer_diag && (p.tsel & ~cur->R)) pend.push_back(i);
              else {
                flush();
                place_diag(i);
              }
              continue;
            }
            const bool starts = (cur->has_perm && ((p.tmask | p.tsel) & cur->touched(K_))) ||
                                popc((u64)(cur->R | p.tmask)) > RB;
            if (starts) {
              fresh();
              flush();  // the waiting diagonal ops open the new phase
            } else {
              flush();
            }
            cur->R |= p.tmask;
            if (C->opt.shm_hoist_dense) {
              // hoist: the dense op joins the earliest dense item of the phase
              // it commutes back to (diagonal runs not acting on its targets,
              // dense items on disjoint bits); the front packing interleaves
              // a layer's single-qubit gates with other gates, which otherwise
              // alternates one-gate dense items with diagonal runs
              int at = (int)cur->items.size();
              for (int k2 = (int)cur->items.size() - 1; k2 >= 0; k2--) {
                const auto &it = cur->items[k2];
                bool conf = false;
                for (int o2 : it.second) {
                  const Pre &q = pre[o2];
                  if (it.first == 1 ? (q.tsel & p.tmask) != 0
                                    : ((q.tmask & (p.tmask | p.tsel)) | (q.tsel & p.tmask)) != 0) {
                    conf = true;
                    break;
                  }
                }
                if (conf) break;
                at = k2;
              }
              int j = -1;
              for (int k2 = at; k2 < (int)cur->items.size(); k2++)
                if (cur->items[k2].first == 0) {
                  j = k2;
                  break;
                }
              if (j >= 0) {
                cur->items[j].second.push_back(i);
                continue;
              }
              if (at < (int)cur->items.size()) {
                cur->items.insert(cur->items.begin() + at, {0, {i}});
                continue;
              }
              cur->diag_open = false;
              cur->items.push_back({0, {i}});
              continue;
            }
            if (cur->diag_open && !(p.tmask & cur->diag_bits)) {
              // commutes with the open diagonal run: execute it first
              const size_t n_it = cur->items.size();
              if (n_it >= 2 && cur->items[n_it - 2].first == 0)
                cur->items[n_it - 2].second.push_back(i);
              else
                cur->items.insert(cur->items.end() - 1, {0, {i}});
            } else {
              cur->diag_open = false;
              if (!cur->items.empty() && cur->items.back().first == 0)
                cur->items.back().second.push_back(i);
              else
                cur->items.push_back({0, {i}});
            }
          }
          flush();
          if (phs.size() > 1 && phs.back().items.empty() && !phs.back().has_perm) phs.pop_back();
          ln.sl.phase_off = (int64_t)C->phases.size();
          ln.sl.ops_off = (int64_t)C->ops.size();
          ln.sl.coef_off = (int64_t)C->coef.size();
          ln.sl.ent_off = (int64_t)C->ents.size();
          ln.sl.term_off = (int64_t)C->terms.size();
          ln.sl.nphase = (int)phs.size();
          auto swzh = [&](u32 j) -> u32 {
            return (u32)(C->dt == ATLAS_C128 ? swz_c128((int)j) : swz_c64((int)j));
          };
          for (PhaseB &pb : phs) {
            int rm = (int)pb.R;
            // fill with the highest free tile bits (keeps low tile bits as lane bits)
            for (int b = K_ - 1; b >= 0 && popc((u64)rm) < RB; b--) rm |= 1 << b;
            ShmPhase ph{};
            int ri = 0;
            int reg_index[16];
            for (int b = 0; b < 16; b++) reg_index[b] = -1;
            for (int b = 0; b < K_; b++)
              if ((rm >> b) & 1) {
                ph.rbit[ri] = b;
                reg_index[b] = ri++;
              }
            for (int i = ri; i < 4; i++) ph.rbit[i] = 0;
            ph.op_begin = (int32_t)(C->ops.size() - ln.sl.ops_off);
            // selector split of one op: register / thread / tile-base parts
            auto split = [&](const Pre &p, int &reg_mask, int &reg_val, ShmOp &op) {
              reg_mask = reg_val = 0;
              for (auto &sv : p.sel) {
                int slot = sv.first, v = sv.second;
                int tb = tile_of_slot[slot];
                if (tb < 0) {
                  op.base_mask |= 1ull << slot;
                  op.base_val |= (u64)v << slot;
                } else if (reg_index[tb] >= 0) {
                  reg_mask |= 1 << reg_index[tb];
                  reg_val |= v << reg_index[tb];
                } else {
                  op.thr_mask |= (uint16_t)(1 << tb);
                  op.thr_val |= (uint16_t)(v << tb);
                }
              }
            };
            auto emit_generic = [&](const Pre &p) {
              ShmOp op{};
              op.type = (uint8_t)p.type;
              if (p.nt >= 1) op.t0 = (uint8_t)reg_index[p.ttile[0]];
              if (p.nt >= 2) op.t1 = (uint8_t)reg_index[p.ttile[1]];
              int reg_mask, reg_val;
              split(p, reg_mask, reg_val, op);
              // element mask over the 2^RB register elements (pair / quad bases
              // for targeted ops: the target bits of e are zero there)
              for (int e = 0; e < (1 << RB); e++)
                if ((e & reg_mask) == reg_val) op.emask |= (uint16_t)(1u << e);
              if (reg_mask == 0 && op.thr_mask == 0 && op.base_mask == 0) op.flags |= OPF_FULL;
              if (p.type == OP_DENSE1) {
                bool real = true;
                for (int i = 0; i < 4; i++)
                  if (p.coef[2 * i + 1] != 0.0) real = false;
                if (real) op.flags |= OPF_REAL;
              }
              op.coef = (int32_t)(C->coef.size() - ln.sl.coef_off);
              for (double d : p.coef) C->coef.push_back(d);
              C->ops.push_back(op);
            };
            for (auto &item : pb.items) {
              if (item.first == 0) {
                for (int i : item.second) emit_generic(pre[i]);
                continue;
              }
              // diagonal run -> factor slots.  A diagonal op multiplies by c
              // where every selector holds; with register selectors (i, vi),
              // (j, vj) the indicator [x_i = vi][x_j = vj] expands into
              // products of F (1), K_i (x_i), K_j (x_j), P_ij (x_i x_j).
              std::map<int, cd> uni;
              std::map<int, std::map<std::tuple<uint16_t, uint16_t, u64, u64>, cd>> cond;
              std::vector<int> generic;
              auto pair_slot = [](int i, int j) {
                static const int tab[4][4] = {{-1, 5, 6, 7}, {5, -1, 8, 9}, {6, 8, -1, 10}, {7, 9, 10, -1}};
                return tab[i][j];
              };
              auto add = [&](int slot, const ShmOp &cnd, cd c) {
                if (cnd.thr_mask == 0 && cnd.base_mask == 0) {
                  auto it = uni.find(slot);
                  if (it == uni.end()) uni[slot] = c;
                  else it->second *= c;
                } else {
                  auto key = std::make_tuple(cnd.thr_mask, cnd.thr_val, cnd.base_mask, cnd.base_val);
                  auto &m = cond[slot];
                  auto it = m.find(key);
                  if (it == m.end()) m[key] = c;
                  else it->second *= c;
                }
              };
              for (int i : item.second) {
                const Pre &p = pre[i];
                if (p.conj) {
                  const cd c(p.coef[0], p.coef[1]);
                  for (auto &mo : p.mono) {
                    ShmOp cnd{};
                    for (auto &sv : p.sel)
                      if (tile_of_slot[sv.first] < 0) {
                        cnd.base_mask |= 1ull << sv.first;
                        cnd.base_val |= (u64)sv.second << sv.first;
                      }
                    // the monomial's own base condition (flips of folded
                    // base-controlled gates); contradictory -> never applies
                    if (((cnd.base_val ^ mo.bv) & cnd.base_mask & mo.bm) != 0) continue;
                    cnd.base_mask |= mo.bm;
                    cnd.base_val |= mo.bv;
                    int rr[2], nr = 0;
                    for (int b = 0; b < K_; b++)
                      if ((mo.m >> b) & 1) {
                        if (reg_index[b] >= 0) rr[nr++] = reg_index[b];
                        else {
                          cnd.thr_mask |= (uint16_t)(1 << b);
                          cnd.thr_val |= (uint16_t)(1 << b);
                        }
                      }
                    const int slot = nr == 0 ? 0 : nr == 1 ? 1 + rr[0] : pair_slot(std::min(rr[0], rr[1]), std::max(rr[0], rr[1]));
                    add(slot, cnd, std::pow(c, mo.e));
                  }
                  continue;
                }
                ShmOp tmp{};
                int reg_mask, reg_val;
                split(p, reg_mask, reg_val, tmp);
                const int nreg = popc((u64)reg_mask);
                if (nreg > 2) {
                  generic.push_back(i);
                  continue;
                }
                const cd c(p.coef[0], p.coef[1]), ci = cd(1) / c;
                std::vector<std::pair<int, cd>> contrib;
                int rb[2], rv[2], nr = 0;
                for (int r = 0; r < RB; r++)
                  if ((reg_mask >> r) & 1) {
                    rb[nr] = r;
                    rv[nr++] = (reg_val >> r) & 1;
                  }
                if (nr == 0) {
                  contrib.push_back({0, c});
                } else if (nr == 1) {
                  if (rv[0]) contrib.push_back({1 + rb[0], c});
                  else {
                    contrib.push_back({0, c});
                    contrib.push_back({1 + rb[0], ci});
                  }
                } else {
                  const int ps = pair_slot(rb[0], rb[1]);
                  if (rv[0] && rv[1]) {
                    contrib.push_back({ps, c});
                  } else if (rv[0] && !rv[1]) {
                    contrib.push_back({1 + rb[0], c});
                    contrib.push_back({ps, ci});
                  } else if (!rv[0] && rv[1]) {
                    contrib.push_back({1 + rb[1], c});
                    contrib.push_back({ps, ci});
                  } else {
                    contrib.push_back({0, c});
                    contrib.push_back({1 + rb[0], ci});
                    contrib.push_back({1 + rb[1], ci});
                    contrib.push_back({ps, c});
                  }
                }
                for (auto &sc : contrib) add(sc.first, tmp, sc.second);
              }
              for (int slot = 0; slot < 11; slot++) {
                auto iu = uni.find(slot);
                auto ic = cond.find(slot);
                cd u = iu == uni.end() ? cd(1) : iu->second;
                bool has_c = ic != cond.end() && !ic->second.empty();
                if (!has_c && std::abs(u - cd(1)) < 1e-15) continue;
                ShmOp op{};
                op.type = OP_DIAG;
                op.t0 = (uint8_t)slot;
                op.coef = (int32_t)(C->coef.size() - ln.sl.coef_off);
                C->coef.push_back(u.real());
                C->coef.push_back(u.imag());
                op.base_mask = (u64)(C->ents.size() - ln.sl.ent_off);
                if (has_c)
                  for (auto &kv : ic->second) {
                    DiagEnt d{};
                    d.thr_mask = std::get<0>(kv.first);
                    d.thr_val = std::get<1>(kv.first);
                    d.base_mask = std::get<2>(kv.first);
                    d.base_val = std::get<3>(kv.first);
                    d.has_base = d.base_mask != 0;
                    d.re = kv.second.real();
                    d.im = kv.second.imag();
                    C->ents.push_back(d);
                  }
                op.base_val = (u64)(C->ents.size() - ln.sl.ent_off);
                C->ops.push_back(op);
              }
              for (int i : generic) emit_generic(pre[i]);
            }
            ph.op_end = (int32_t)(C->ops.size() - ln.sl.ops_off);
            ph.term_begin = ph.term_end = (int32_t)(C->terms.size() - ln.sl.term_off);
            if (pb.has_perm && !pb.aff_identity(K_)) {
              // merge the tile-base terms: [b = 0] v = v ^ [b = 1] v, and terms
              // with equal conditions XOR together (<= one per non-active bit
              // for CX chains controlled by non-active qubits)
              {
                std::map<std::pair<u64, u64>, u32> mt;
                for (auto &t : pb.terms) {
                  u64 bm = std::get<0>(t), bv = std::get<1>(t);
                  u32 v = std::get<2>(t);
                  if (popc(bm) == 1 && bv == 0) {
                    pb.c0 ^= v;
                    bv = bm;
                  }
                  mt[{bm, bv}] ^= v;
                }
                pb.terms.clear();
                for (auto &kv : mt)
                  if (kv.second) pb.terms.push_back(std::make_tuple(kv.first.first, kv.first.second, kv.second));
              }
              ph.permuted = 1;
              for (int b = 0; b < 16; b++) ph.colimg[b] = b < K_ ? (uint16_t)swzh(pb.col[b]) : 0;
              ph.c0_swz = swzh(pb.c0);
              for (auto &t : pb.terms) {
                PermTerm pt{};
                pt.base_mask = std::get<0>(t);
                pt.base_val = std::get<1>(t);
                pt.vec_swz = swzh(std::get<2>(t));
                u32 v = std::get<2>(t);
                for (int b = 0; b < K_; b++)
                  if ((v >> b) & 1) pt.gvec |= 1ull << act[b];
                C->terms.push_back(pt);
              }
              ph.term_end = (int32_t)(C->terms.size() - ln.sl.term_off);
            }
            {
              // lanes of one shared-memory wavefront (thread bits 0..W-1):
              // pick W non-register tile bits whose swizzled bank groups are
              // independent for the gather (identity addresses) and for the
              // permuted store (images colimg); default ascending order
              // when it already is conflict-free
              const int W = C->dt == ATLAS_C128 ? 3 : 4;
              const u32 wm = (1u << W) - 1;
              std::vector<int> nr;
              for (int b = 0; b < K_; b++)
                if (!((rm >> b) & 1)) nr.push_back(b);
              auto rank_of = [&](const std::vector<u32> &vs) {
                u32 basis[16] = {0};
                int r = 0;
                for (u32 v : vs) {
                  for (int bit = 15; bit >= 0 && v; bit--)
                    if ((v >> bit) & 1) {
                      if (!basis[bit]) {
                        basis[bit] = v;
                        r++;
                        v = 0;
                      } else {
                        v ^= basis[bit];
                      }
                    }
                }
                return r;
              };
              auto cost = [&](const std::vector<int> &sel) {
                std::vector<u32> ld, st;
                for (int b : sel) {
                  ld.push_back(swzh(1u << b) & wm);
                  st.push_back((ph.permuted ? (u32)ph.colimg[b] : swzh(1u << b)) & wm);
                }
                return (1 << (W - rank_of(ld))) + (1 << (W - rank_of(st)));
              };
              ph.qlane = 0xffff;
              if ((int)nr.size() >= W) {
                std::vector<int> def(nr.begin(), nr.begin() + W);
                int best = cost(def);
                std::vector<int> bsel;
                const int nn = (int)nr.size();
                for (u32 m = 0; m < (1u << nn) && best > 2; m++) {
                  if (popc((u64)m) != W) continue;
                  std::vector<int> sel;
                  for (int i = 0; i < nn; i++)
                    if ((m >> i) & 1) sel.push_back(nr[i]);
                  const int c = cost(sel);
                  if (c < best) {
                    best = c;
                    bsel = sel;
                  }
                }
                if (!bsel.empty()) {
                  u32 q = 0xffff;
                  for (int i = 0; i < W; i++) q = (q & ~(15u << (4 * i))) | ((u32)bsel[i] << (4 * i));
                  ph.qlane = (uint16_t)q;
                }
              }
            }
            C->phases.push_back(ph);
          }
          if (sl == 0) C->kplans[k].kernels[&K - &kp.kernels[0]].nphase = (int)phs.size();
          {
            // direct HBM store of the last phase when its register bits
            // avoid the 5 lowest tile bits (lanes = tile bits 0..4)
            const ShmPhase &lp = C->phases.back();
            const PhaseB &lb = phs.back();
            int rm = 0;
            for (int i = 0; i < RB; i++) rm |= 1 << lp.rbit[i];
            const int lowm = (1 << std::min(5, K_ - RB)) - 1;
            const bool perm = lp.permuted != 0;
            auto dep = [&](u32 x) {
              u64 r = 0;
              for (int b = 0; b < K_; b++)
                if ((x >> b) & 1) r |= 1ull << act[b];
              return r;
            };
            // the 32 lanes of a warp must write one contiguous 512-B run:
            // tile bits 0..4 are physical slots 0..4 and the folded map sends
            // them into that span (it is invertible, so onto it)
            bool coalesced = K_ - RB >= 5 && dep(0x1fu) == 0x1full;
            if (perm)
              for (int b = 0; b < 5 && coalesced; b++)
                if (lb.col[b] & ~0x1fu) coalesced = false;
            ln.sl.last_direct = C->opt.shm_direct_store && !(rm & lowm) && coalesced;
            // the direct store needs lanes = tile bits 0..4 in order
            if (ln.sl.last_direct) C->phases.back().qlane = 0xffff;
            for (int b = 0; b < 16; b++)
              ln.sl.lcol[b] = b < K_ ? dep(perm ? lb.col[b] : (1u << b)) : 0;
            ln.sl.lc0 = perm ? dep(lb.c0) : 0;
          }
          ln.sl.nops = (int)(C->ops.size() - ln.sl.ops_off);
          ln.sl.ncoef = (int)(C->coef.size() - ln.sl.coef_off);
          ln.sl.nent = (int)(C->ents.size() - ln.sl.ent_off);
          ln.sl.nterm = (int)(C->terms.size() - ln.sl.term_off);
        }
        C->prog[sl].push_back(ln);
      }
      if (!scalar_done) {
        Launch ln;
        ln.type = L_SCALE;
        ln.stage = k;
        ln.sre = scalar[sl].real();
        ln.sim = scalar[sl].imag();
        ln.bytes = pass_bytes;
        C->prog[sl].push_back(ln);
      }
      // fuse the next remap's pack (a bit permutation of the local slots)
      // into this stage's last shared-memory launch: it stores its output
      // permuted into the other buffer, so the standalone pack pass
      // (a full read + write of the shard) disappears (P:L1312 Shard,
      // north_star (4))
      if (C->opt.shm_fuse_pack && !C->opt.inplace_remap && k + 1 < s && !SW[k + 1].pre[sl].empty() &&
          SW[k + 1].pre[sl][0].type == L_PACK && !C->prog[sl].empty() &&
          C->prog[sl].back().type == L_SHM && C->prog[sl].back().stage == k) {
        Launch &last = C->prog[sl].back();
        last.sl.out_perm_off = SW[k + 1].pre[sl][0].newpos_off;
        last.newpos_off = last.sl.out_perm_off;
        SW[k + 1].pre[sl].erase(SW[k + 1].pre[sl].begin());
      } else if (C->opt.shm_fuse_pack && C->opt.shm_fuse_exchange && !C->opt.inplace_remap && !C->offload &&
                 k + 1 < s && C->exch[k + 1].gp > 0 && C->exch[k + 1].gp <= 3 &&
                 (SW[k + 1].pre[sl].empty() || SW[k + 1].pre[sl][0].type != L_PACK) && !C->prog[sl].empty() &&
                 C->prog[sl].back().type == L_SHM && C->prog[sl].back().stage == k) {
        // a remap without a pack: the identity "pack", so that the launch
        // can carry the exchange below
        Launch &last = C->prog[sl].back();
        last.sl.out_perm_off = (int64_t)C->newpos.size();
        last.newpos_off = last.sl.out_perm_off;
        for (int b = 0; b < C->L; b++) C->newpos.push_back(b);
      }
    }
    // ... and the exchange itself: when every slot's last launch of the
    // stage carries the fused pack, those launches store each packed block
    // straight into the buffer of the rank it goes to (peer memory over
    // NVLink, CUDA IPC; another slot's buffer in a virtual world), so no
    // separate all-to-all runs (north_star (4); P:L1312 Shard).  All slots
    // or none: a rank's stores land in its peers' buffers.
    if (C->opt.shm_fuse_exchange && !C->offload && k + 1 < s && C->exch[k + 1].gp > 0 &&
        C->exch[k + 1].gp <= 3) {
      bool all = true;
      for (int sl = 0; sl < C->nslots; sl++) {
        const auto &P = C->prog[sl];
        if (P.empty() || P.back().type != L_SHM || P.back().stage != k || P.back().sl.out_perm_off < 0)
          all = false;
      }
      if (all)
        for (int sl = 0; sl < C->nslots; sl++) C->prog[sl].back().sl.peer_gp = C->exch[k + 1].gp;
    }
  }
  C->planned = true;
  C->blobs_ready = false;
  C->jit_ready = false;
  C->plan_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
}

// ------------------------------------------------------------------ JSON
static void jmask(std::ostringstream &o, u64 m) {
  o << "[";
  bool first = true;
  for (int q = 0; q < 64; q++)
    if ((m >> q) & 1) {
      if (!first) o << ",";
      o << q;
      first = false;
    }
  o << "]";
}

std::string plan_json(const atlas_ctx *C) {
  std::ostringstream o;
  o << "{\"n\":" << C->n << ",\"L\":" << C->L << ",\"G\":" << C->G << ",\"R\":0"
    << ",\"c\":" << C->c << ",\"dtype\":\"" << (C->dt == ATLAS_C128 ? "c128" : "c64") << "\""
    << ",\"staging\":{\"s\":" << C->sp.s << ",\"cost\":" << C->sp.cost
    << ",\"exact\":" << (C->sp.exact ? "true" : "false") << ",\"gate_stage\":[";
  for (size_t g = 0; g < C->sp.gate_stage.size(); g++) o << (g ? "," : "") << C->sp.gate_stage[g];
  o << "]},\"cost_model\":\"" << C->cm.source << "\",\"K_tile\":" << C->K_tile
    << ",\"ls_qubits\":" << C->cm.ls_qubits << ",\"stages\":[";
  for (int k = 0; k < C->sp.s; k++) {
    if (k) o << ",";
    o << "{\"local\":";
    jmask(o, C->sp.local[k]);
    o << ",\"global\":";
    jmask(o, C->sp.global[k]);
    o << ",\"regional\":";
    jmask(o, (C->n == 64 ? ~0ull : ((1ull << C->n) - 1)) & ~C->sp.local[k] & ~C->sp.global[k]);
    o << ",\"sigma\":[";
    for (int q = 0; q < C->n; q++) o << (q ? "," : "") << C->maps[k].sigma[q];
    o << "],\"flip_begin\":[";
    for (int q = 0; q < C->n; q++) o << (q ? "," : "") << C->maps[k].flip_begin[q];
    o << "],\"flip_end\":[";
    for (int q = 0; q < C->n; q++) o << (q ? "," : "") << C->maps[k].flip_end[q];
    o << "],\"packed\":" << (k > 0 && C->exch[k].packed ? "true" : "false");
    {
      bool xf = false;  // the exchange rides on the previous stage's last launch
      if (!C->prog.empty())
        for (const Launch &ln : C->prog[0])
          if (ln.stage == k - 1 && ln.type == L_SHM && ln.sl.peer_gp > 0) xf = true;
      o << ",\"exchange_fused\":" << (xf ? "true" : "false");
    }
    o << ",\"pack_fused\":";
    {
      int64_t off = -1;
      bool fused = false;
      if (!C->prog.empty())
        for (const Launch &ln : C->prog[0]) {
          if (ln.stage == k && ln.type == L_PACK) off = ln.newpos_off;
          if (ln.stage == k - 1 && ln.type == L_SHM && ln.newpos_off >= 0 && C->exch[k].packed) {
            off = ln.newpos_off;
            fused = true;
          }
        }
      o << (fused ? "true" : "false") << ",\"pack_newpos\":";
      if (off < 0) {
        o << "null";
      } else {
        o << "[";
        for (int i = 0; i < C->L; i++) o << (i ? "," : "") << C->newpos[off + i];
        o << "]";
      }
    }
    o << ",\"remap_qubits\":" << (k > 0 ? C->exch[k].gp : 0);
    o << ",\"gates\":[";
    for (size_t i = 0; i < C->stage_gates[k].size(); i++) o << (i ? "," : "") << C->stage_gates[k][i];
    o << "],\"kernel_cost\":" << C->kplans[k].total << ",\"kernels\":[";
    for (size_t i = 0; i < C->kplans[k].kernels.size(); i++) {
      const Kernel &K = C->kplans[k].kernels[i];
      if (i) o << ",";
      o << "{\"kind\":\"" << (K.kind == K_FUSION ? "fusion" : "shm") << "\",\"cost\":" << K.cost
        << ",\"phases\":" << K.nphase
        << ",\"qubits\":";
      jmask(o, K.qubits);
      o << ",\"gates\":[";
      for (size_t j = 0; j < K.gates.size(); j++) o << (j ? "," : "") << K.gates[j];
      o << "]}";
    }
    o << "]}";
  }
  o << "],\"plan_us\":" << C->plan_us << "}";
  return o.str();
}

}  // namespace atlas
