// jit.cpp -- plan-specialised shared-memory kernels (NVRTC, sm_100a).
//
// PAPER.md P:L1964 defines a shared-memory kernel as "load a micro-batch into
// shared memory and apply the gates one by one".  The generic shm_kernel in
// kernels.cu interprets the lowered op program (ShmOp/ShmPhase/DiagEnt/
// PermTerm, device.h) for every tile: per op it loads a header, dispatches
// on the op type and the target register bit, and loads the coefficients.
// The circuit is fixed once atlas_plan returns, so this file turns the SAME
// lowered program into straight-line CUDA for each launch: phases unrolled,
// targets and element masks compile-time, gate coefficients literal constants,
// permutation ops register renames, tile/thread conditions plain branches.
// The generated kernel computes exactly what the interpreter computes (same
// tile, phases, op order and arithmetic per element), so the interpreter
// stays the reference for the JIT path in the GPU parity tests (option
// shm_jit = 0 selects it).
//
// NVRTC is loaded at run time (libnvrtc.so.12 from the CUDA toolkit of this
// image); the cubin is loaded with cudaLibraryLoadData.  Identical sources
// are compiled once per process.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <cmath>
#include <complex>
#include <map>
#include <random>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ctx.h"

namespace atlas {

// ------------------------------------------------------------------- NVRTC
namespace {
typedef int nvrtcResult_;
typedef void *nvrtcProgram_;
struct NvrtcApi {
  void *h = nullptr;
  nvrtcResult_ (*create)(nvrtcProgram_ *, const char *, const char *, int, const char *const *,
                         const char *const *) = nullptr;
  nvrtcResult_ (*compile)(nvrtcProgram_, int, const char *const *) = nullptr;
  nvrtcResult_ (*cubinSize)(nvrtcProgram_, size_t *) = nullptr;
  nvrtcResult_ (*cubin)(nvrtcProgram_, char *) = nullptr;
  nvrtcResult_ (*logSize)(nvrtcProgram_, size_t *) = nullptr;
  nvrtcResult_ (*log)(nvrtcProgram_, char *) = nullptr;
  nvrtcResult_ (*destroy)(nvrtcProgram_ *) = nullptr;
  const char *(*err)(nvrtcResult_) = nullptr;
};
NvrtcApi g_nvrtc;
std::mutex g_nvrtc_mu;

void nvrtc_load() {
  std::lock_guard<std::mutex> lk(g_nvrtc_mu);
  if (g_nvrtc.h) return;
  const char *names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  for (const char *nm : names) {
    g_nvrtc.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    if (g_nvrtc.h) break;
  }
  if (!g_nvrtc.h)
    fail(ATLAS_E_CUDA, "cannot load libnvrtc.so.12 (needed by shm_jit=1): %s", dlerror());
  auto S = [](const char *n) {
    void *p = dlsym(g_nvrtc.h, n);
    if (!p) fail(ATLAS_E_CUDA, "libnvrtc lacks %s", n);
    return p;
  };
  g_nvrtc.create = (decltype(g_nvrtc.create))S("nvrtcCreateProgram");
  g_nvrtc.compile = (decltype(g_nvrtc.compile))S("nvrtcCompileProgram");
  g_nvrtc.cubinSize = (decltype(g_nvrtc.cubinSize))S("nvrtcGetCUBINSize");
  g_nvrtc.cubin = (decltype(g_nvrtc.cubin))S("nvrtcGetCUBIN");
  g_nvrtc.logSize = (decltype(g_nvrtc.logSize))S("nvrtcGetProgramLogSize");
  g_nvrtc.log = (decltype(g_nvrtc.log))S("nvrtcGetProgramLog");
  g_nvrtc.destroy = (decltype(g_nvrtc.destroy))S("nvrtcDestroyProgram");
  g_nvrtc.err = (decltype(g_nvrtc.err))S("nvrtcGetErrorString");
}

struct JitEntry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int smem = 0, nt = 0, attr_set = 0, threads = 0;
  bool zero_ok = false;
  // TMA tile loads: the tensor dimensions the kernel was generated for
  // (runs of local slots: start, length, active low bits)
  int tma_rank = 0;
  int tstart[5] = {0}, tlen[5] = {0}, tabits[5] = {0};
  // device copies of the encoded tensor map, one per state buffer the kernel
  // has read (written once; distinct addresses, so no descriptor cached for
  // one map is ever looked up for another)
  std::map<const void *, void *> dmaps;
};
std::mutex g_cache_mu;
std::unordered_map<std::string, JitEntry *> g_cache;  // source -> compiled kernel

// --------------------------------------------------------------- emitter
// fp64 coefficient pool of the kernel being generated: SASS DFMA/DMUL take a
// 32-bit immediate at most, so a general double literal costs two UMOVs into
// a uniform register pair before every use; a __constant__ table entry is
// read as a c[bank][offset] operand with no extra instruction (measured on
// su2random n=28: UMOV was 18% of the issued instructions of the heaviest
// shared-memory kernel).  Values whose low 32 bits are zero (+-1, 0.5, ...)
// stay immediates.
struct LitPool {
  std::vector<double> vals;
  std::map<uint64_t, int> index;
};
thread_local LitPool *g_pool = nullptr;

// fp64 complex factors of diagonal-run elements, read from a shared-memory
// table (option shm_lit_smem): a uniform-address LDS.128 per element replaces
// the four UMOVs that materialise the two literals in uniform registers
// (UMOV was 24% of the issued instructions of su2random's heaviest kernel).
// ptxas cannot hoist the loads out of the tile loop (the loop's shared stores
// may alias the table), so no register is held across tiles.
struct LitTab {
  std::vector<std::pair<double, double>> vals;
  std::map<std::pair<uint64_t, uint64_t>, int> index;
  int intern(double re, double im) {
    uint64_t a, b;
    memcpy(&a, &re, 8);
    memcpy(&b, &im, 8);
    auto it = index.find({a, b});
    if (it != index.end()) return it->second;
    const int k = (int)vals.size();
    vals.push_back({re, im});
    index[{a, b}] = k;
    return k;
  }
};
thread_local LitTab *g_ltab = nullptr;

std::string lit(double d, bool f32) {
  char b[64];
  if (f32) {
    float f = (float)d;
    if (f == 0.0f) return "0.0f";
    snprintf(b, sizeof b, "(%af)", (double)f);
  } else {
    if (d == 0.0) return "0.0";
    uint64_t bits;
    memcpy(&bits, &d, 8);
    if (g_pool && (bits & 0xffffffffull) != 0) {
      auto it = g_pool->index.find(bits);
      int k;
      if (it != g_pool->index.end()) {
        k = it->second;
      } else {
        k = (int)g_pool->vals.size();
        g_pool->vals.push_back(d);
        g_pool->index[bits] = k;
      }
      snprintf(b, sizeof b, "KC[%d]", k);
      return b;
    }
    snprintf(b, sizeof b, "(%a)", d);
  }
  return b;
}

std::string u64lit(uint64_t v) {
  char b[32];
  snprintf(b, sizeof b, "0x%llxull", (unsigned long long)v);
  return b;
}

// y = M x over D register elements idx[0..D-1] (row-major complex M), the
// terms ordered as in the interpreter (column by column), zero entries
// dropped.
void emit_block(std::ostringstream &o, int D, const int *idx, const double *m, bool f32,
                const char *ind) {
  o << ind << "{\n";
  for (int c = 0; c < D; c++) o << ind << "  const T x" << c << " = v[" << idx[c] << "];\n";
  for (int r = 0; r < D; r++) {
    for (int part = 0; part < 2; part++) {
      // part 0: re = sum mr*x.x - mi*x.y ; part 1: im = sum mr*x.y + mi*x.x
      std::string acc;
      for (int c = 0; c < D; c++) {
        const double mr = m[2 * (r * D + c)], mi = m[2 * (r * D + c) + 1];
        const double k0 = mr, k1 = part == 0 ? -mi : mi;
        const std::string x0 = "x" + std::to_string(c) + (part == 0 ? ".x" : ".y");
        const std::string x1 = "x" + std::to_string(c) + (part == 0 ? ".y" : ".x");
        const std::pair<double, std::string> terms[2] = {{k0, x0}, {k1, x1}};
        for (auto &t : terms) {
          if (t.first == 0.0) continue;
          if (acc.empty()) acc = lit(t.first, f32) + " * " + t.second;
          else acc = "fma(" + lit(t.first, f32) + ", " + t.second + ", " + acc + ")";
        }
      }
      if (acc.empty()) acc = f32 ? "0.0f" : "0.0";
      o << ind << "  v[" << idx[r] << "]." << (part == 0 ? "x" : "y") << " = " << acc << ";\n";
    }
  }
  o << ind << "}\n";
}

void emit_cmul_lit(std::ostringstream &o, int e, double re, double im, bool f32, const char *ind) {
  if (re == 1.0 && im == 0.0) return;
  if (im == 0.0) {
    o << ind << "v[" << e << "].x *= " << lit(re, f32) << "; v[" << e << "].y *= " << lit(re, f32)
      << ";\n";
    return;
  }
  if (g_ltab && !f32 && re != 0.0) {
    const int k = g_ltab->intern(re, im);
    o << ind << "{ const T f = lt[" << k << "]; const T a = v[" << e << "]; v[" << e
      << "].x = f.x * a.x - f.y * a.y; v[" << e << "].y = f.x * a.y + f.y * a.x; }\n";
    return;
  }
  o << ind << "{ const T a = v[" << e << "]; v[" << e << "].x = " << lit(re, f32) << " * a.x - "
    << lit(im, f32) << " * a.y; v[" << e << "].y = " << lit(re, f32) << " * a.y + " << lit(im, f32)
    << " * a.x; }\n";
}

const int kDiagSel[11] = {0, 1, 2, 4, 8, 3, 5, 9, 6, 10, 12};

}  // namespace

int shm_nbuf_effective(int dtype, const ShmLaunch &sl);
size_t shm_jit_smem(const std::string &src);
void shm_jit_prime(void *jit);

// TMA tile loads (option shm_tma, fp64 pipe kernels).  The shard is viewed
// as a tensor of at most 5 dimensions, each a run of consecutive local slots
// whose low part is active (covered by the box) and whose high part is
// non-active (selected by the tile's coordinates): dim 0 = slots 0..2 (8
// amplitudes = 16 doubles = one 128-B swizzle row), then greedy runs of at
// most 8 active slots followed by the non-active slots up to the next
// active one.  One cp.async.bulk.tensor per tile moves all 2^K amplitudes
// into shared memory with the 128-B swizzle (16-B chunk index ^= row index
// mod 8, i.e. tile index j -> j ^ ((j >> 3) & 7)), completing on the tile's
// mbarrier.  Launches whose active slots need more than 5 runs, or do not
// include slots 0..2, keep the per-thread cp.async gather.
struct TmaDims {
  int rank = 0;
  int start[5], len[5], abits[5];
};
static bool tma_dims(const ShmLaunch &sl, TmaDims &d) {
  const int L = sl.K + __builtin_popcountll(sl.nonactive);
  uint64_t act = 0;
  for (int b = 0; b < sl.K; b++) act |= 1ull << sl.act[b];
  if ((act & 7) != 7 || sl.K < 6) return false;
  d.rank = 1;
  d.start[0] = 0;
  d.len[0] = 3;
  d.abits[0] = 3;
  int cur = 3;
  while (cur < L) {
    if (d.rank == 5) return false;
    const int s0 = cur;
    int a = 0;
    while (cur < L && ((act >> cur) & 1) && a < 8) {
      cur++;
      a++;
    }
    while (cur < L && !((act >> cur) & 1)) cur++;
    if (cur - s0 > 31) return false;
    d.start[d.rank] = s0;
    d.len[d.rank] = cur - s0;
    d.abits[d.rank] = a;
    d.rank++;
  }
  return true;
}
thread_local bool g_no_tma = false;
thread_local int g_force_pipe = -1;  // autotune: -1 = the option, 0/1 = forced
thread_local int g_force_ld = -1;    // autotune: 0 = no direct last-phase store
struct TmaRetry {};

// The straight-line source of one shared-memory launch (same skeleton as
// kernels.cu shm_kernel: ring of tile buffers filled with cp.async, register
// phases, permuted stores, optional direct HBM store of the last phase).
static std::string shm_jit_source_body(const atlas_ctx *C, const ShmLaunch &sl, const std::string &name);

// The shared-memory literal table (shm_lit_smem) goes after every other
// shared buffer of the launch; its entries are known only once the body is
// generated, so the table, its fill loop and the size are patched in here.
// A launch whose table does not fit beside its resident CTAs falls back to
// literals.
static std::string patch_lit_table(const std::string &body, const LitTab &tab) {
  auto drop = [&](std::string s) {
    for (const char *ph : {"//@LT_DECL@\n", "//@LT_FILL@\n"}) {
      const size_t at = s.find(ph);
      if (at != std::string::npos) s.erase(at, strlen(ph));
    }
    return s;
  };
  if (tab.vals.empty()) return drop(body);
  const size_t smem = shm_jit_smem(body);
  const size_t lt_off = (smem + 15) & ~(size_t)15;
  const size_t nsmem = lt_off + 16 * tab.vals.size();
  int bt = 0, minb = 1;
  {
    const char *p = strstr(body.c_str(), "__launch_bounds__(");
    if (p) sscanf(p, "__launch_bounds__(%d, %d)", &bt, &minb);
  }
  const size_t cap = minb >= 2 ? 233472 / minb - 1024 : 232448;
  if (nsmem > cap) return std::string();
  std::string s = body;
  auto rep = [&](const std::string &from, const std::string &to) {
    const size_t at = s.find(from);
    if (at == std::string::npos) fail(ATLAS_E_CUDA, "shm_jit: literal table placeholder missing");
    s.replace(at, from.size(), to);
  };
  std::ostringstream t;
  t << "#define LT_OFF " << lt_off << "\n__constant__ double2 LTC[" << tab.vals.size() << "] = {";
  char b[96];
  for (size_t i = 0; i < tab.vals.size(); i++) {
    snprintf(b, sizeof b, "%s{%a, %a}", i ? ", " : "", tab.vals[i].first, tab.vals[i].second);
    t << b;
  }
  t << "};\n#define SMEM_BYTES " << nsmem << "\n";
  rep("#define SMEM_BYTES " + std::to_string(smem) + "\n", t.str());
  rep("//@LT_DECL@\n", "  T *lt = reinterpret_cast<T *>(smraw + LT_OFF);\n");
  rep("//@LT_FILL@\n", "  for (int i = threadIdx.x; i < " + std::to_string(tab.vals.size()) +
                           "; i += BLOCK_THREADS) lt[i] = LTC[i];\n");
  return s;
}

std::string shm_jit_source(const atlas_ctx *C, const ShmLaunch &sl, const std::string &name) {
  LitPool pool;
  const bool use_pool = C->dt == ATLAS_C128 && C->opt.shm_const_pool;
  g_pool = use_pool ? &pool : nullptr;
  LitTab tab;
  const bool use_tab = C->dt == ATLAS_C128 && C->opt.shm_lit_smem && !use_pool;
  std::string body;
  try {
    g_ltab = use_tab ? &tab : nullptr;
    g_no_tma = false;
    try {
      body = shm_jit_source_body(C, sl, name);
    } catch (const TmaRetry &) {  // TMA needs the pipe pipeline; it was not chosen
      g_no_tma = true;
      tab = LitTab();
      pool = LitPool();
      body = shm_jit_source_body(C, sl, name);
    }
    g_ltab = nullptr;
    std::string patched = patch_lit_table(body, tab);
    if (patched.empty()) {  // the table does not fit: literals
      pool = LitPool();
      body = patch_lit_table(shm_jit_source_body(C, sl, name), LitTab());
      g_no_tma = false;
    } else {
      body = patched;
    }
  } catch (...) {
    g_pool = nullptr;
    g_ltab = nullptr;
    g_no_tma = false;
    throw;
  }
  g_pool = nullptr;
  if (pool.vals.empty()) return body;
  // the table goes after the header comment and typedefs (before the kernel)
  std::ostringstream t;
  t << "__constant__ double KC[" << pool.vals.size() << "] = {";
  char b[64];
  for (size_t i = 0; i < pool.vals.size(); i++) {
    snprintf(b, sizeof b, "%s%a", i ? ", " : "", pool.vals[i]);
    t << b;
  }
  t << "};\n";
  const size_t at = body.find("#define SMEM_BYTES");
  return body.substr(0, at) + t.str() + body.substr(at);
}

static std::string shm_jit_source_body(const atlas_ctx *C, const ShmLaunch &sl, const std::string &name) {
  const bool f32 = C->dt == ATLAS_C64;
  const int K = sl.K, RB = sl.RB, NT = 1 << (K - RB), NE = 1 << RB, TILE = 1 << K;
  const int nbuf = shm_nbuf_effective(f32 ? 1 : 0, sl);
  const int esz = f32 ? 8 : 16;
  const ShmOp *ops = C->ops.data() + sl.ops_off;
  const double *coef = C->coef.data() + sl.coef_off;
  const ShmPhase *ph = C->phases.data() + sl.phase_off;
  const DiagEnt *ents = C->ents.data() + sl.ent_off;
  const PermTerm *terms = C->terms.data() + sl.term_off;
  // fused remap pack (plan.cpp): the launch writes its output to the other
  // buffer with every local slot b moved to slot np[b] -- the bit
  // permutation of the pack that precedes the next stage's exchange
  // (P:L1312 Shard).  P() maps an output offset; being a bit permutation it
  // distributes over the XOR / OR of disjoint offsets, so every store-side
  // constant is mapped at generation time and the tile base by a table.
  const bool operm = sl.out_perm_off >= 0;
  // fused exchange: the packed output goes to the destination ranks' buffers
  const int pgp = operm ? sl.peer_gp : 0;
  const int PSH = C->L - pgp;
  std::vector<int> np;
  if (operm) np.assign(C->newpos.begin() + sl.out_perm_off, C->newpos.begin() + sl.out_perm_off + C->L);
  auto PB = [&](uint64_t x) {
    if (!operm) return x;
    uint64_t r = 0;
    for (int b = 0; b < (int)np.size(); b++)
      if ((x >> b) & 1) r |= 1ull << np[b];
    return r;
  };
  int minb = (nbuf == 1 && (K - RB) >= 8 && (K - RB) <= 9 && (esz << K) <= 65536) ? 2 : 1;

  // ---- shared-memory swizzles per phase boundary and lanes per phase.
  // A swizzle is S(j) = j ^ sum_{b >= W} j_b * col[b] (col[b] < 2^W): linear,
  // an involution, and the identity on the W lowest tile bits (the lanes of
  // the cp.async load and of the copy-out).  Phase p gathers from the layout
  // of boundary p-1 and stores into that of boundary p; the layout of the
  // first load is the global swizzle (device.h).  A permuted phase may pick a
  // new layout for its store so that both its store and the next phase's
  // gather hit W independent bank groups (for the 8 / 16 lanes of one
  // wavefront) where the global swizzle cannot.
  const int W = f32 ? 4 : 3;
  const unsigned WM = (1u << W) - 1;
  typedef std::vector<unsigned> Swz;
  std::vector<Swz> swzs(1, Swz(K, 0));
  for (int b = W; b < K; b++) swzs[0][b] = 1u << (b % W);
  // the lowering (plan.cpp) stores its tile vectors under the global swizzle
  // GL (device.h); the layout of the tile load (swzs[0]) is GL for the
  // cp.async gather, the 128-B TMA swizzle for TMA loads
  const Swz GL = swzs[0];
  TmaDims tdim;
  const bool tma = !f32 && nbuf == 1 && C->opt.shm_tma && C->opt.shm_pipe && !g_no_tma &&
                   (1 << (K - RB)) * 2 <= 512 && tma_dims(sl, tdim);
  if (tma)
    for (int b = W; b < K; b++) swzs[0][b] = b < 2 * W ? 1u << (b - W) : 0u;
  auto Sx = [&](const Swz &c, unsigned j) {
    unsigned r = j;
    for (int b = W; b < K; b++)
      if ((j >> b) & 1) r ^= c[b];
    return r;
  };
  auto rank_w = [&](const std::vector<unsigned> &vs) {
    unsigned basis[16] = {0};
    int r = 0;
    for (unsigned v : vs) {
      v &= WM;
      for (int bit = W - 1; bit >= 0 && v; bit--)
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
  // unswizzled folded map of each permuted phase (the lowering stores it
  // under the global swizzle, an involution)
  std::vector<std::vector<unsigned>> Acol(sl.nphase);
  std::vector<unsigned> Ac0(sl.nphase, 0);
  for (int p = 0; p < sl.nphase; p++)
    if (ph[p].permuted) {
      Acol[p].resize(K);
      for (int b = 0; b < K; b++) Acol[p][b] = Sx(GL, ph[p].colimg[b]);
      Ac0[p] = Sx(GL, ph[p].c0_swz);
    }
  const int lastp = sl.nphase - 1;
  const bool ld_ = sl.last_direct != 0 && g_force_ld != 0;
  // fold0: a leading phase with no op but its folded permutation (a CX
  // block whose dense gates come later) only moves the tile through shared
  // memory once more; its permuted store is folded into the tile load
  // instead -- every cp.async writes its element straight to the permuted
  // (and re-swizzled) position -- and the phase is not emitted (option
  // shm_fold_perm; cp.async loads only, not when the phase's gather feeds a
  // direct HBM store)
  const bool fold0 = C->opt.shm_fold_perm && nbuf == 1 && !tma && !sl.zfill_cap && sl.nphase >= 1 && ph[0].permuted &&
                     ph[0].op_begin == ph[0].op_end && !(ld_ && lastp == 0);
  std::vector<int> rmask(sl.nphase), gsw(sl.nphase, 0), ssw(sl.nphase, 0);
  std::vector<unsigned> qln(sl.nphase, 0xffff);
  for (int p = 0; p < sl.nphase; p++) {
    int m = 0;
    for (int i = 0; i < RB; i++) m |= 1 << ph[p].rbit[i];
    rmask[p] = m;
  }
  auto subsets = [&](int p) {
    // candidate lane sets: the lowering's choice, the default, then all
    std::vector<std::vector<int>> out;
    std::vector<int> nr;
    for (int b = 0; b < K; b++)
      if (!((rmask[p] >> b) & 1)) nr.push_back(b);
    if ((int)nr.size() < W) return out;
    if (ph[p].qlane != 0xffff) {
      std::vector<int> q;
      for (int i = 0; i < W; i++) q.push_back((ph[p].qlane >> (4 * i)) & 15);
      out.push_back(q);
    }
    out.push_back(std::vector<int>(nr.begin(), nr.begin() + W));
    const int nn = (int)nr.size();
    for (unsigned mm = 0; mm < (1u << nn); mm++) {
      if (__builtin_popcount(mm) != W) continue;
      std::vector<int> q;
      for (int i = 0; i < nn; i++)
        if ((mm >> i) & 1) q.push_back(nr[i]);
      out.push_back(q);
    }
    return out;
  };
  auto gather_rank = [&](const std::vector<int> &sub, const Swz &G) {
    std::vector<unsigned> v;
    for (int b : sub) v.push_back(Sx(G, 1u << b));
    return rank_w(v);
  };
  auto store_rank = [&](int p, const std::vector<int> &sub, const Swz &T) {
    std::vector<unsigned> v;
    for (int b : sub) v.push_back(Sx(T, Acol[p][b]));
    return rank_w(v);
  };
  auto enc = [&](const std::vector<int> &sub) {
    unsigned q = 0xffff;
    for (int i = 0; i < (int)sub.size(); i++) q = (q & ~(15u << (4 * i))) | ((unsigned)sub[i] << (4 * i));
    return q;
  };
  std::mt19937 rng(12345u);  // deterministic: identical on every rank
  bool fold_ok = false;
  if (fold0) {
    // the load writes with lanes = tile bits 0..W-1 (8 / 16 consecutive
    // threads): find a layout under which those lanes' permuted images hit
    // W bank groups and the next phase can gather conflict-free
    std::vector<int> ll;
    for (int b = 0; b < W; b++) ll.push_back(b);
    for (int trial = 0; trial < 400 && !fold_ok; trial++) {
      Swz T(K, 0);
      if (trial == 0) T = swzs[0];
      else
        for (int b = W; b < K; b++) T[b] = rng() & WM;
      if (store_rank(0, ll, T) != W) continue;
      bool next_ok = sl.nphase == 1;
      if (!next_ok)
        for (auto &s2 : subsets(1))
          if (gather_rank(s2, T) == W) {
            next_ok = true;
            break;
          }
      if (!next_ok) continue;
      int ti = -1;
      for (size_t i = 0; i < swzs.size(); i++)
        if (swzs[i] == T) ti = (int)i;
      if (ti < 0) {
        ti = (int)swzs.size();
        swzs.push_back(T);
      }
      qln[0] = enc(ll);
      ssw[0] = ti;
      if (sl.nphase > 1) gsw[1] = ti;
      fold_ok = true;
    }
  }
  for (int p = fold_ok ? 1 : 0; p < sl.nphase; p++) {
    const Swz G = swzs[gsw[p]];
    const auto subs = subsets(p);
    if (subs.empty()) continue;
    if (ld_ && p == lastp) {  // direct store: lanes = tile bits 0..4
      ssw[p] = gsw[p];
      continue;
    }
    const bool perm = ph[p].permuted != 0;
    const bool swz_free = C->opt.shm_swz_phase != 0;
    // best gather-only choice (fallback)
    std::vector<int> best = subs[0];
    int bestr = -1;
    for (auto &sub : subs) {
      const int r = gather_rank(sub, G) + (perm ? store_rank(p, sub, G) : W);
      if (r > bestr) {
        bestr = r;
        best = sub;
      }
    }
    qln[p] = enc(best);
    ssw[p] = gsw[p];
    if (p + 1 < sl.nphase) gsw[p + 1] = gsw[p];
    if (!perm || !swz_free || bestr == 2 * W) continue;
    // a permuted phase whose store conflicts: look for a store layout
    bool done = false;
    for (int trial = 0; trial < 400 && !done; trial++) {
      Swz T(K, 0);
      if (trial == 0) T = swzs[0];
      else
        for (int b = W; b < K; b++) T[b] = rng() & WM;
      for (auto &sub : subs) {
        if (gather_rank(sub, G) != W || store_rank(p, sub, T) != W) continue;
        // the next phase must find a conflict-free gather under T
        bool next_ok = p + 1 >= sl.nphase;
        if (!next_ok)
          for (auto &s2 : subsets(p + 1))
            if (gather_rank(s2, T) == W) {
              next_ok = true;
              break;
            }
        if (!next_ok) continue;
        int ti = -1;
        for (size_t i = 0; i < swzs.size(); i++)
          if (swzs[i] == T) ti = (int)i;
        if (ti < 0) {
          ti = (int)swzs.size();
          swzs.push_back(T);
        }
        qln[p] = enc(sub);
        ssw[p] = ti;
        if (p + 1 < sl.nphase) gsw[p + 1] = ti;
        done = true;
        break;
      }
    }
  }
  if (getenv("ATLAS_DEBUG_SWZ"))
    for (int p = 0; p < sl.nphase; p++) {
      std::vector<int> sub;
      if (qln[p] != 0xffff)
        for (int i = 0; i < W; i++) sub.push_back((qln[p] >> (4 * i)) & 15);
      else
        for (int b = 0; b < K && (int)sub.size() < W; b++)
          if (!((rmask[p] >> b) & 1)) sub.push_back(b);
      fprintf(stderr, "swz phase %d perm %d gather %d store %d layouts %d/%d\n", p, (int)ph[p].permuted,
              gather_rank(sub, swzs[gsw[p]]),
              ph[p].permuted && !(ld_ && p == lastp) ? store_rank(p, sub, swzs[ssw[p]]) : W, gsw[p], ssw[p]);
    }
  // distinct thread-index tables: (register mask, lanes, gather layout) ->
  // jt and its gather address; (register mask, lanes, store images) -> the
  // permuted store address
  std::vector<int> jslot(sl.nphase), sslot(sl.nphase, -1);
  std::vector<std::pair<long long, int>> jmasks;  // (mask | lanes << 16, layout)
  std::vector<std::pair<int, std::vector<uint16_t>>> smaps;
  std::vector<std::vector<uint16_t>> simg(sl.nphase);
  for (int p = 0; p < sl.nphase; p++) {
    const int key = rmask[p] | ((int)qln[p] << 16);
    int js = -1;
    for (size_t i = 0; i < jmasks.size(); i++)
      if (jmasks[i].first == key && jmasks[i].second == gsw[p]) js = (int)i;
    if (js < 0) {
      js = (int)jmasks.size();
      jmasks.push_back({key, gsw[p]});
    }
    jslot[p] = js;
    if (ph[p].permuted) {
      std::vector<uint16_t> img(K);
      for (int b = 0; b < K; b++) img[b] = (uint16_t)Sx(swzs[ssw[p]], Acol[p][b]);
      simg[p] = img;
      int ss = -1;
      for (size_t i = 0; i < smaps.size(); i++)
        if (smaps[i].first == key && smaps[i].second == img) ss = (int)i;
      if (ss < 0) {
        ss = (int)smaps.size();
        smaps.push_back({key, img});
      }
      sslot[p] = ss;
    }
  }
  // tile-base deposit tables: one 256-entry table per byte of the tile index
  int tbits = 0;
  while ((1ull << tbits) < sl.ntiles) tbits++;
  const int nbt = std::max(1, (tbits + 7) / 8);
  // base-only conditional factors of diagonal slots (conditions on
  // non-active qubits only: uniform over a tile) are evaluated once per tile
  // by one designated thread per slot into a double-buffered SMEM table
  // instead of by every thread
  std::map<int, int> bslot;  // op index -> base-factor slot
  for (int q = 0; q < sl.nops; q++) {
    const ShmOp &dq = ops[q];
    if (dq.type != OP_DIAG) continue;
    bool any = false;
    for (int i = (int)dq.base_mask; i < (int)dq.base_val; i++)
      if (ents[i].thr_mask == 0 && ents[i].has_base) any = true;
    if (any) {
      const int k = (int)bslot.size();
      bslot[q] = k;
    }
  }
  const int NB = (int)bslot.size();
  // thread-only conditional factors (conditions on the thread's tile bits
  // only): constant per thread, computed once in the prologue into a
  // per-thread SMEM table (<= 32 KiB per CTA)
  std::map<int, int> tslot;   // op index -> thread-factor slot
  std::map<int, int> op_phase;
  for (int p = 0; p < sl.nphase; p++)
    for (int q = ph[p].op_begin; q < ph[p].op_end; q++) op_phase[q] = p;
  if (C->opt.shm_tfac_min > 0)
    for (int q = 0; q < sl.nops; q++) {
      const ShmOp &dq = ops[q];
      if (dq.type != OP_DIAG) continue;
      int cnt = 0;
      for (int i = (int)dq.base_mask; i < (int)dq.base_val; i++)
        if (ents[i].thr_mask != 0 && !ents[i].has_base) cnt++;
      // a table load replaces cnt compare-and-multiply steps
      const bool any = cnt >= C->opt.shm_tfac_min;
      if (any && (size_t)(tslot.size() + 1) * NT * esz <= 32768) {
        const int k = (int)tslot.size();
        tslot[q] = k;
      }
    }
  int NTF = (int)tslot.size();
  size_t off_bfac = 0, off_tfac = 0;
  auto layout = [&](int ntile_bufs, size_t &oj, size_t &os, size_t &ob, size_t &om) {
    oj = (size_t)ntile_bufs * TILE * esz;
    os = oj + (size_t)jmasks.size() * NT * 4;
    ob = (os + (size_t)smaps.size() * NT * 2 + 15) & ~(size_t)15;
    om = ob + (size_t)nbt * 256 * 8 * (operm ? 2 : 1);
    off_bfac = (om + 6 * 8 + 15) & ~(size_t)15;
    off_tfac = off_bfac + (size_t)4 * NB * esz;
    return off_tfac + (size_t)NTF * NT * esz;  // bfac: [group][parity][slot]
  };
  size_t off_jtab, off_stab, off_btab, off_mbar;
  // pipe: one CTA of two thread groups (each a full tile's worth of
  // threads, named barriers) sharing a ring of three tile buffers: a tile's
  // load is issued into the buffer the other group just finished with, so up
  // to two loads are in flight while both groups compute; completion is
  // tracked by cp.async -> mbarrier arrivals.  The k-th tile of the CTA
  // (buffer k % 3) completes on mbarrier k % 6, not k % 3: consecutive
  // phases of one mbarrier then belong to tiles of the SAME group (k and
  // k + 6), so a group never waits on phase j + 1 of a barrier whose phase j
  // (the other group's tile) is still in flight -- with k % 3, a parity wait
  // for phase j + 1 succeeds while phase j is incomplete (try_wait.parity
  // only distinguishes the current phase from the preceding one), which let
  // a fast group read a buffer before its load landed (round-1 qsvm n=28
  // mirror, |a0 - 1| = 2e-6).
  // (two groups of 256: the fp64 2^12 tiles; fp32's 2 x 512 threads at 64
  // registers measured slower than two single-buffer CTAs)
  bool pipe = nbuf == 1 && (g_force_pipe >= 0 ? g_force_pipe != 0 : C->opt.shm_pipe != 0) && 2 * NT <= 512 &&
              layout(3, off_jtab, off_stab, off_btab, off_mbar) + 1024 <= 233472;
  if (tma && !pipe) throw TmaRetry();
  // the thread-factor table must not cost occupancy (or exceed the opt-in
  // limit): drop slots until it fits beside the resident CTAs
  if (pipe) minb = 1;
  if (NTF) {
    const int keep = NTF;
    NTF = 0;
    const size_t base_sz = layout(pipe ? 3 : nbuf, off_jtab, off_stab, off_btab, off_mbar);
    const size_t cap = (minb >= 2 ? 233472 / minb - 1024 : 232448) - (tma ? 1024 : 0);
    const size_t fit = base_sz < cap ? (cap - base_sz) / ((size_t)NT * esz) : 0;
    NTF = (int)std::min<size_t>(keep, fit);
    for (auto it = tslot.begin(); it != tslot.end();)
      it = it->second >= NTF ? tslot.erase(it) : std::next(it);
  }
  // TMA: 1 KiB of slack so the tile buffers can start on a 1024-B boundary
  // (the 128-B swizzle pattern repeats every 1024 B of shared address)
  const size_t smem = layout(pipe ? 3 : nbuf, off_jtab, off_stab, off_btab, off_mbar) + (tma ? 1024 : 0);
  const int BT = pipe ? 2 * NT : NT;  // threads per CTA
  // option shm_ctas = 3: three resident CTAs per SM (register cap 80) when
  // their shared memory fits the SM
  if (minb == 2 && C->opt.shm_ctas >= 3 && 3 * (smem + 1024) <= 233472) minb = 3;

  std::ostringstream o;
  o << "// generated by jit.cpp: shared-memory kernel, K=" << K << " RB=" << RB
    << " phases=" << sl.nphase << " ops=" << sl.nops << "\n";
  o << "typedef unsigned long long u64; typedef unsigned int u32; typedef unsigned short u16;\n";
  o << (f32 ? "typedef float R; typedef float2 T;\n" : "typedef double R; typedef double2 T;\n");
  o << "#define SMEM_BYTES " << smem << "\n";
  if (pgp) o << "#define ATLAS_PEER " << pgp << "\nstruct PeerTab { T *p[8]; };\n";
  if (tma) {
    o << "#define ATLAS_TMA " << tdim.rank;
    for (int d = 0; d < tdim.rank; d++) o << " " << tdim.start[d] << ":" << tdim.len[d] << ":" << tdim.abits[d];
    o << "\nstruct __align__(64) TMap { unsigned long long v[16]; };\n";
  }
  // zmode (early pipeline only): 1 = the input is all zeros, 2 = the input
  // is |0...0> on this rank (atlas_run's initial state): the first tile
  // load is synthesised in registers and nothing is read from HBM
  o << "#define ZERO_OK " << (nbuf == 1 && !fold_ok ? 1 : 0) << "\n";
  if (fold_ok) o << "// phase 0 (a permutation only) folded into the tile load\n";
  o << "__device__ __forceinline__ u64 pdep64(u64 v, u64 mask) { u64 r = 0; while (mask) { u64 lo = "
       "mask & (~mask + 1); if (v & 1) r |= lo; v >>= 1; mask ^= lo; } return r; }\n";
  o << "#define BLOCK_THREADS " << BT << "\n";
  if (pipe) {
    o << "__device__ __forceinline__ void gsync(int g) { asm volatile(\"bar.sync %0, " << NT
      << ";\" :: \"r\"(1 + g) : \"memory\"); }\n";
    // a tile load that never lands (a broken tensor map, a lost arrival)
    // traps after ~10 s instead of hanging the device
    o << "__device__ __forceinline__ void mbar_wait(unsigned a, unsigned par) { unsigned ok = 0; "
         "const long long t0 = clock64(); do { "
         "asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 "
         "%0, 1, 0, p; }\" : \"=r\"(ok) : \"r\"(a), \"r\"(par) : \"memory\"); "
         "if (!ok && clock64() - t0 > 20000000000ll) __trap(); } while (!ok); }\n";
  }
  o << "extern \"C\" __global__ void __launch_bounds__(" << BT << ", " << minb << ") " << name
    << "(T *__restrict__ st, T *dst, int zmode, u64 nact, u32 ntl, u32 zfill"
    << (tma ? ", const TMap *__restrict__ tmg" : "") << (pgp ? ", const PeerTab ptab" : "") << ") {\n";
  if (pgp) o << "  __shared__ T *pts[8];\n";
  if (tma) {
    o << "  extern __shared__ __align__(1024) unsigned char smraw_[];\n";
    o << "  const unsigned smpad = (1024u - ((unsigned)__cvta_generic_to_shared(smraw_) & 1023u)) & 1023u;\n";
    o << "  unsigned char *smraw = smraw_ + smpad;\n";
    if (getenv("ATLAS_DEBUG_ALIGN"))
      o << "  if (threadIdx.x == 0 && smpad) printf(\"atlas: block %d dynamic smem base %% 1024 = %u\\n\", "
           "(int)blockIdx.x, 1024u - smpad);\n";
  } else {
    o << "  extern __shared__ __align__(16) unsigned char smraw[];\n";
  }
  o << "  T *buf = reinterpret_cast<T *>(smraw);\n";
  o << "//@LT_DECL@\n";
  o << "  u32 *jtab = reinterpret_cast<u32 *>(smraw + " << off_jtab << ");\n";
  o << "  u16 *stab = reinterpret_cast<u16 *>(smraw + " << off_stab << ");\n";
  o << "  u64 *btab = reinterpret_cast<u64 *>(smraw + " << off_btab << ");\n";
  if (NB) o << "  T *bfac = reinterpret_cast<T *>(smraw + " << off_bfac << ");\n  int itp = 0;\n";
  if (pipe) {
    o << "  const int tid = threadIdx.x & " << NT - 1 << ", grp = threadIdx.x / " << NT << ";\n";
    o << "  const unsigned mbar0 = (unsigned)__cvta_generic_to_shared(smraw + " << off_mbar << ");\n";
    // TMA: one arrival (with the transaction bytes) per tile; cp.async: one
    // per thread of the group
    o << "  if (threadIdx.x == 0) { for (int i = 0; i < 6; i++) asm volatile(\"mbarrier.init.shared::cta.b64 "
         "[%0], %1;\" :: \"r\"(mbar0 + 8 * i), \"r\"(" << (tma ? 1 : NT) << ") : \"memory\");"
      << (tma ? " asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");" : "") << " }\n";
  } else {
    o << "  const int tid = threadIdx.x;\n";
  }
  // tile-base deposit tables
  // nact (launch argument): the non-active slots the tiles run over -- all of
  // them, or fewer when the caller knows the tiles with a 1 on some of them
  // hold zeros in and out (runtime.cu, zero-support tracking); ntl = 2^|nact|
  o << "  for (int i = threadIdx.x; i < " << nbt * 256 << "; i += " << BT << ") { const int c = i >> 8; u64 m = "
    << "nact; for (int k = 0; k < 8 * c && m; k++) m &= m - 1; btab[i] = "
    << "pdep64((u64)(i & 255), m); }\n";
  if (operm) {
    o << "  u64 *obtab = btab + " << nbt * 256 << ";\n";
    o << "  for (int i = threadIdx.x; i < " << nbt * 256 << "; i += " << BT << ") { const u64 x = btab[i]; u64 r = 0;";
    for (int b = 0; b < (int)np.size(); b++)
      if (sl.nonactive >> b & 1) o << " r |= ((x >> " << b << ") & 1ull) << " << np[b] << ";";
    o << " obtab[i] = r; }\n";
  }
  // per-thread tile indices of every distinct (register mask, lane order):
  // thread bit i -> tile bit order[i] (kernels.cu shm_kernel prologue)
  auto thread_order = [&](int key) {
    const int m = key & 0xffff, q = (key >> 16) & 0xffff;
    std::vector<int> ord;
    int used = m;
    if (q != 0xffff)
      for (int i = 0; i < 4; i++) {
        const int nb = (q >> (4 * i)) & 15;
        if (nb == 15) break;
        ord.push_back(nb);
        used |= 1 << nb;
      }
    for (int b = 0; b < K; b++)
      if (!((used >> b) & 1)) ord.push_back(b);
    return ord;
  };
  if (pipe) o << "  if (grp == 0) {\n";
  for (size_t js = 0; js < jmasks.size(); js++) {
    o << "  { int jt = 0; u32 sj = 0;";
    const std::vector<int> ord = thread_order((int)jmasks[js].first);
    const Swz &G = swzs[jmasks[js].second];
    for (size_t t = 0; t < ord.size(); t++)
      o << " if ((tid >> " << t << ") & 1) { jt |= " << (1 << ord[t]) << "; sj ^= " << Sx(G, 1u << ord[t])
        << "u; }";
    o << " jtab[" << js * NT << " + tid] = (sj << 16) | (u32)jt; }\n";
  }
  for (size_t ss = 0; ss < smaps.size(); ss++) {
    o << "  { u32 sa = 0;";
    const std::vector<int> ord = thread_order(smaps[ss].first);
    for (size_t t = 0; t < ord.size(); t++)
      o << " if ((tid >> " << t << ") & 1) sa ^= " << smaps[ss].second[ord[t]] << "u;";
    o << " stab[" << ss * NT << " + tid] = (u16)sa; }\n";
  }
  if (pipe) o << "  }\n";
  if (NTF) {
    o << "  T *tfac = reinterpret_cast<T *>(smraw + " << off_tfac << ");\n";
    if (pipe) o << "  if (grp == 0) {\n";
    for (auto &kv : tslot) {
      const ShmOp &dq = ops[kv.first];
      const int p = op_phase[kv.first];
      o << "  { const int jt = (int)(jtab[" << jslot[p] * NT << " + tid] & 0xffffu); R fx = 1, fy = 0;\n";
      for (int i = (int)dq.base_mask; i < (int)dq.base_val; i++) {
        const DiagEnt &d = ents[i];
        if (!(d.thr_mask != 0 && !d.has_base)) continue;
        o << "    if ((jt & " << d.thr_mask << ") == " << d.thr_val << ") { const R nx = fx * "
          << lit(d.re, f32) << " - fy * " << lit(d.im, f32) << "; fy = fx * " << lit(d.im, f32)
          << " + fy * " << lit(d.re, f32) << "; fx = nx; }\n";
      }
      o << "    tfac[" << kv.second * NT << " + tid].x = fx; tfac[" << kv.second * NT << " + tid].y = fy; }\n";
    }
    if (pipe) o << "  }\n";
  }
  // this thread's HBM offset inside a tile
  o << "  u64 off_t = 0;";
  for (int i = 0; i < K - RB; i++) o << " if ((tid >> " << i << ") & 1) off_t |= " << u64lit(1ull << sl.act[i]) << ";";
  if (operm) {
    o << "\n  u64 ooff_t = 0;";
    for (int i = 0; i < K - RB; i++) o << " if ((tid >> " << i << ") & 1) ooff_t |= " << u64lit(PB(1ull << sl.act[i])) << ";";
  }
  // load destination of this thread's elements: the load layout, or (fold0)
  // the permuted, re-swizzled position phase 0 would have stored them at
  auto ldimg = [&](unsigned j) {
    if (!fold_ok) return Sx(swzs[0], j);
    unsigned r = 0;
    for (int b = 0; b < K; b++)
      if ((j >> b) & 1) r ^= simg[0][b];
    return r;
  };
  o << "\n  int sw_tid = 0;";
  for (int t = 0; t < K - RB; t++) o << " if ((tid >> " << t << ") & 1) sw_tid ^= " << ldimg(1u << t) << ";";
  o << "\n";
  // copy-out reads the layout of the last boundary
  const Swz &SO = swzs[ssw[lastp]];
  o << "  int sw_out = 0;";
  for (int t = 0; t < K - RB; t++) o << " if ((tid >> " << t << ") & 1) sw_out ^= " << Sx(SO, 1u << t) << ";";
  o << "\n";
  o << "  const unsigned sm_base = (unsigned)__cvta_generic_to_shared(buf);\n";
  o << "//@LT_FILL@\n";
  if (pgp) o << "  if (threadIdx.x < " << (1 << pgp) << ") pts[threadIdx.x] = ptab.p[threadIdx.x];\n";
  o << "  __syncthreads();\n";
  // fused exchange: the destination blocks in shared memory (a run-time
  // index into the parameter array would go through local memory); a
  // store picks its block once per tile from the bits of its offset that
  // are uniform over the tile and thread, XOR / OR the element's constant
  // high bits
  if (pgp) o << "  T *const *ptab_s = reinterpret_cast<T *const *>(pts);\n";
  o << "  auto tile_base = [&](u64 tile) { return btab[tile & 255]";
  for (int c = 1; c < nbt; c++) o << " | btab[" << 256 * c << " + ((tile >> " << 8 * c << ") & 255)]";
  o << "; };\n";
  if (operm) {
    o << "  auto otile_base = [&](u64 tile) { return obtab[tile & 255]";
    for (int c = 1; c < nbt; c++) o << " | obtab[" << 256 * c << " + ((tile >> " << 8 * c << ") & 255)]";
    o << "; };\n";
  }
  // per-register-element offsets (constant)
  std::vector<uint64_t> itoff(NE);
  for (int it = 0; it < NE; it++) {
    uint64_t x = 0;
    for (int i = 0; i < RB; i++)
      if ((it >> i) & 1) x |= 1ull << sl.act[K - RB + i];
    itoff[it] = x;
  }
  o << "  auto issue_load = [&](int bsel, " << (pipe ? "int msel, " : "") << "u64 base) {\n    const T *g = st + base + off_t;\n";
  if (fold_ok) {
    // phase 0's constant and tile-dependent offsets (the folded map's
    // translation and its CX controlled by non-active qubits)
    o << "    int swl = sw_tid ^ " << Sx(swzs[ssw[0]], Ac0[0]) << ";\n";
    for (int i = ph[0].term_begin; i < ph[0].term_end; i++)
      o << "    if ((base & " << u64lit(terms[i].base_mask) << ") == " << u64lit(terms[i].base_val)
        << ") swl ^= " << Sx(swzs[ssw[0]], Sx(GL, terms[i].vec_swz)) << ";\n";
  } else {
    o << "    const int swl = sw_tid;\n";
  }
  // lazy zeros: elements the first gather takes as zero need no load; the
  // warp-uniform and element parts of that test skip whole cp.async
  // instructions without per-thread state (the gather's per-element test
  // covers the rest)
  // (fp64 only: fp32 kernels have no register to spare at the 64 cap)
  const bool zskip_ld = sl.zfill_cap && !f32;
  if (zskip_ld) o << "    const bool zw = ((unsigned)tid & ~31u & zfill) != 0u;\n";
  for (int it = 0; it < NE; it++) {
    if (zskip_ld) o << "    if (!zw && !(" << (it << (K - RB)) << "u & zfill))";
    o << "    { const unsigned sa = sm_base + (unsigned)((bsel * " << TILE << " + (swl ^ "
      << ldimg((unsigned)(it * NT)) << ")) * " << esz << "); const T *ga = g + " << u64lit(itoff[it])
      << "; ";
    if (!f32) o << "asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\\n\" ::\"r\"(sa), \"l\"(ga)); }\n";
    else o << "asm volatile(\"cp.async.ca.shared.global [%0], [%1], 8;\\n\" ::\"r\"(sa), \"l\"(ga)); }\n";
  }
  if (pipe)
    o << "    asm volatile(\"cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\" :: \"r\"(mbar0 + 8 * msel) : \"memory\");\n  };\n";
  else
    o << "    asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\");\n  };\n";
  // pipe, zero mode: the ring protocol without data (plain arrivals)
  if (pipe && !tma)
    o << "  auto issue = [&](int bsel, int msel, u64 base) { if (!zmode) issue_load(bsel, msel, base); else asm volatile("
         "\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(mbar0 + 8 * msel) : \"memory\"); };\n";
  if (tma) {
    // one thread of the group: the tile's coordinates from its base, one
    // bulk tensor copy completing on the tile's mbarrier (expect_tx)
    // the tensor map lives in global memory, one per (kernel, state buffer),
    // written once by the host: acquire it for the tensormap proxy before
    // the first bulk tensor copy of this CTA
    o << "  const u64 tmap_a = reinterpret_cast<u64>(tmg);\n";
    o << "  if (tid == 0) asm volatile(\"fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\" :: \"l\"(tmap_a) : \"memory\");\n";
    o << "  auto issue = [&](int bsel, int msel, u64 base) {\n    if (tid != 0) return;\n"
      << "    const unsigned mb_ = mbar0 + 8 * msel;\n"
      << "    if (zmode) { asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(mb_) : \"memory\"); return; }\n"
      << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
      << "    asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(mb_), \"r\"("
      << (TILE * esz) << ") : \"memory\");\n";
    o << "    const int c0 = 0";
    for (int d = 1; d < tdim.rank; d++)
      o << ", c" << d << " = (int)((base >> " << tdim.start[d] << ") & " << u64lit((1ull << tdim.len[d]) - 1) << ")";
    o << ";\n";
    o << "    asm volatile(\"cp.async.bulk.tensor." << tdim.rank
      << "d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {";
    for (int d = 0; d < tdim.rank; d++) o << (d ? ", " : "") << "%" << (2 + d);
    o << "}], [%" << (2 + tdim.rank) << "];\" :: \"r\"(sm_base + (unsigned)bsel * " << (TILE * esz)
      << "u), \"l\"(tmap_a)";
    for (int d = 0; d < tdim.rank; d++) o << ", \"r\"(c" << d << ")";
    o << ", \"r\"(mb_) : \"memory\");\n  };\n";
  }
  const std::string GS = pipe ? "gsync(grp);" : "__syncthreads();";
  // tb[x ^ a] for one thread part x and the element constants a of a phase:
  // when x's set bits above the bank bits (W) never meet a's (x and a are
  // images of disjoint tile-bit sets), x ^ a = (x ^ (a & WM)) + (a & ~WM),
  // so one pointer per distinct low part serves every element and each
  // access is an LDS/STS with an immediate offset (option shm_addr_split;
  // otherwise the XOR and the scaling are recomputed per element).
  const bool asplit = C->opt.shm_addr_split != 0;
  int agroup = 0;
  auto addr_group = [&](const std::string &x, const std::vector<int> &as, const char *ind) {
    std::vector<std::string> out;
    if (!asplit) {
      for (int a : as) out.push_back("tb[" + x + " ^ " + std::to_string(a) + "]");
      return out;
    }
    std::map<int, std::string> ptr;
    for (int a : as) {
      const int lo = a & (int)WM, hi = a & ~(int)WM;
      auto it = ptr.find(lo);
      if (it == ptr.end()) {
        const std::string nm = "q" + std::to_string(agroup++);
        o << ind << "T *" << nm << " = tb + (" << x << " ^ " << lo << ");\n";
        it = ptr.emplace(lo, nm).first;
      }
      out.push_back(it->second + "[" + std::to_string(hi) + "]");
    }
    return out;
  };

  const int last = sl.nphase - 1;
  const bool ld = ld_;
  if (ld) {
    o << "  u64 gthr = 0;\n  { const int jtl = (int)(jtab[" << jslot[last] * NT << " + tid] & 0xffffu);";
    for (int b = 0; b < K; b++)
      if (sl.lcol[b]) o << " if ((jtl >> " << b << ") & 1) gthr ^= " << u64lit(PB(sl.lcol[b])) << ";";
    o << " }\n";
  }
  if (pipe) {
    o << "  const u64 G = gridDim.x;\n";
    o << "  if ((u64)blockIdx.x >= " << "ntl" << ") return;\n";
  } else {
    o << "  u64 tile = blockIdx.x;\n  if (tile >= " << "ntl" << ") return;\n";
    o << "  const u64 G = gridDim.x;\n";
  }
  // early = one tile buffer: the next tile's load is issued as soon as every
  // thread has read the current tile out of shared memory for the last time
  // (the last phase's gather, or the copy-out), so it overlaps the last
  // phase's arithmetic and the HBM stores; the other CTA of the SM covers
  // the rest.
  const bool early = nbuf == 1;
  const std::string NTL = "ntl";
  const std::string next_issue =
      pipe ? "{ const u64 nx = blockIdx.x + (u64)(i + 3) * G; if (nx < " + NTL + ") issue(b, mb < 3 ? mb + 3 : mb - 3, tile_base(nx)); }"
           : "if (!zmode) { const u64 nx = tile + G; if (nx < " + NTL + ") issue_load(0, tile_base(nx)); }";
  // zero tiles (zmode): the input of this launch is |0...0> on this rank
  // (zmode 2) or all zeros (zmode 1), so every tile except tile 0 of rank 0
  // holds zeros; every op of the launch is linear and keeps a tile inside its
  // own tile (a shared-memory kernel touches active qubits only), so such a
  // tile's output is exactly zero: it is stored as zeros with none of the
  // phases (one write-only pass instead of a full compute pass).  The pipe
  // ring still gets its arrival for tile i + 3.
  std::string zero_tile;
  {
    std::ostringstream z;
    // zmode bit 2 (lazy zeros, runtime.cu): the zero tiles are not even
    // stored -- every later launch that reads them zero-fills them (zfill)
    // until a launch has rewritten the whole shard
    z << "    if (zmode && ((zmode & 3) == 1 || tile != 0)) {\n";
    z << "      if (!(zmode & 4)) {\n";
    z << "      T zz; zz.x = 0; zz.y = 0;\n";
    if (pgp) {
      z << "      const u64 gy = obase + ooff_t;\n";
      std::map<uint64_t, int> blk;
      for (int it = 0; it < NE; it++) {
        const uint64_t c = PB(itoff[it]) >> PSH;
        if (!blk.count(c)) {
          const int k = (int)blk.size();
          blk[c] = k;
          z << "      T *zd" << k << " = ptab_s[(int)(gy >> " << PSH << ") | " << c << "] + (gy & "
            << u64lit((1ull << PSH) - 1) << "); __builtin_assume(__isGlobal(zd" << k << "));\n";
        }
      }
      for (int it = 0; it < NE; it++)
        z << "      zd" << blk[PB(itoff[it]) >> PSH] << "[" << u64lit(PB(itoff[it]) & ((1ull << PSH) - 1))
          << "] = zz;\n";
    } else {
      z << (operm ? "      T *g = dst + obase + ooff_t;\n" : "      T *g = st + base + off_t;\n");
      for (int it = 0; it < NE; it++) z << "      g[" << u64lit(PB(itoff[it])) << "] = zz;\n";
    }
    z << "      }\n";
    if (pipe) z << "      " << next_issue << "\n";
    if (NB) z << "      itp ^= 1;\n";
    z << "      continue;\n    }\n";
    zero_tile = z.str();
  }
  if (pipe) {
    // tiles i = 0, 1, 2 of this CTA's sequence into buffers 0, 1, 2, each
    // issued by the group that will process it (i & 1)
    o << "  for (int i = grp; i < 3; i += 2) { const u64 t = blockIdx.x + (u64)i * G; if (t < " << NTL
      << ") issue(i, i, tile_base(t)); }\n";
  } else if (early) {
    o << "  if (!zmode) issue_load(0, tile_base(tile));\n";
  } else {
    for (int k = 0; k < nbuf - 1; k++)
      o << "  { const u64 t = tile + " << k << "ull * G; if (t < " << NTL
        << ") issue_load(" << k << ", tile_base(t)); else asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\"); }\n";
  }
  if (pipe) {
    o << "  int mb = grp;  // i % 6 (i: the CTA's tile counter; mbarrier of tile i)\n";
    o << "  for (unsigned i = grp;; i += 2, mb = mb >= 4 ? mb - 4 : mb + 2) {\n";
    o << "    const u64 tile = blockIdx.x + (u64)i * G;\n    if (tile >= " << NTL << ") break;\n";
    o << "    const u64 base = tile_base(tile);\n";
    if (operm) o << "    const u64 obase = otile_base(tile);\n";
    o << "    const int b = mb < 3 ? mb : mb - 3;\n";
    o << "    mbar_wait(mbar0 + 8 * mb, (i / 6) & 1);\n";
    o << zero_tile;
  } else {
  o << "  int b = 0;\n";
  o << "  for (; tile < " << NTL << "; tile += G) {\n";
  o << "    const u64 base = tile_base(tile);\n";
  if (operm) o << "    const u64 obase = otile_base(tile);\n";
  if (early) o << zero_tile;
  const int nwarps = BT / 32;
  for (auto &kv : bslot) {
    const int bk = kv.second;
    const ShmOp &dq = ops[kv.first];
    const int desig = (bk % nwarps) * 32 + (bk / nwarps) % 32;
    o << "    if (threadIdx.x == " << desig << ") { R fx = 1, fy = 0;\n";
    for (int i = (int)dq.base_mask; i < (int)dq.base_val; i++) {
      const DiagEnt &d = ents[i];
      if (!(d.thr_mask == 0 && d.has_base)) continue;
      o << "      if ((base & " << u64lit(d.base_mask) << ") == " << u64lit(d.base_val)
        << ") { const R nx = fx * " << lit(d.re, f32) << " - fy * " << lit(d.im, f32) << "; fy = fx * "
        << lit(d.im, f32) << " + fy * " << lit(d.re, f32) << "; fx = nx; }\n";
    }
    o << "      bfac[itp * " << NB << " + " << bk << "].x = fx; bfac[itp * " << NB << " + " << bk
      << "].y = fy; }\n";
  }
  }
  if (pipe && NB) {
    // per group: its own double-buffered table, a designated thread of the
    // group, and a group barrier before the factors are read
    const int gw = NT / 32;
    for (auto &kv : bslot) {
      const int bk = kv.second;
      const ShmOp &dq = ops[kv.first];
      const int desig = (bk % gw) * 32 + (bk / gw) % 32;
      o << "    if (tid == " << desig << ") { R fx = 1, fy = 0;\n";
      for (int i = (int)dq.base_mask; i < (int)dq.base_val; i++) {
        const DiagEnt &d = ents[i];
        if (!(d.thr_mask == 0 && d.has_base)) continue;
        o << "      if ((base & " << u64lit(d.base_mask) << ") == " << u64lit(d.base_val)
          << ") { const R nx = fx * " << lit(d.re, f32) << " - fy * " << lit(d.im, f32) << "; fy = fx * "
          << lit(d.im, f32) << " + fy * " << lit(d.re, f32) << "; fx = nx; }\n";
      }
      o << "      bfac[(grp * 2 + itp) * " << NB << " + " << bk << "].x = fx; bfac[(grp * 2 + itp) * " << NB
        << " + " << bk << "].y = fy; }\n";
    }
    o << "    gsync(grp);\n";
  }
  if (pipe) {
  } else if (early) {
    o << "    asm volatile(\"cp.async.wait_group 0;\\n\" ::: \"memory\");\n";
  } else {
    o << "    { const u64 far = tile + " << (nbuf - 1) << "ull * G; const int fb = (b + " << (nbuf - 1)
      << ") % " << nbuf << "; if (far < " << NTL
      << ") issue_load(fb, tile_base(far)); else asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\");"
      << " asm volatile(\"cp.async.wait_group " << (nbuf - 1) << ";\\n\" ::: \"memory\"); }\n";
  }
  if (!pipe) o << "    __syncthreads();\n";
  o << "    T *tb = buf + b * " << TILE << ";\n";
  o << "    T v[" << NE << "];\n";
  double pend = 1.0;  // deferred uniform scalar (sign blocks)
  const bool defer_scalar = C->opt.shm_defer_scalar != 0;
  for (int p = fold_ok ? 1 : 0; p < sl.nphase; p++) {
    const ShmPhase &P = ph[p];
    int sr[4] = {0, 0, 0, 0};
    for (int i = 0; i < RB; i++) sr[i] = (int)Sx(swzs[gsw[p]], 1u << P.rbit[i]);
    o << "    { // phase " << p << "\n";
    o << "      const u32 jj = jtab[" << jslot[p] * NT << " + tid]; const int jt = (int)(jj & 0xffffu); "
      << "const int sj = (int)(jj >> 16); (void)jt;\n";
    {
      std::vector<int> as(NE, 0);
      for (int e = 0; e < NE; e++)
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) as[e] ^= sr[i];
      if (sl.zfill_cap && p == 0) o << "      const unsigned zt = (unsigned)jt & zfill;\n";
      if (early && p == 0) {
        o << "      if (zmode) {\n";
        for (int e2 = 0; e2 < NE; e2++) o << "        v[" << e2 << "].x = 0; v[" << e2 << "].y = 0;\n";
        o << "        if ((zmode & 3) == 2 && tile == 0 && jt == 0) v[0].x = 1;\n      } else {\n";
      }
      const auto ax = addr_group("sj", as, "      ");
      if (sl.zfill_cap && p == 0) {
        // lazy zeros (zfill, launch argument: tile bits of active qubits
        // still |0>): an element with such a bit set is taken as zero --
        // the shard holds no zeros there, only what earlier runs left
        for (int e = 0; e < NE; e++) {
          unsigned eb = 0;
          for (int i = 0; i < RB; i++)
            if ((e >> i) & 1) eb |= 1u << P.rbit[i];
          o << "      if (zt | (" << eb << "u & zfill)) { v[" << e << "].x = 0; v[" << e << "].y = 0; } else v[" << e
            << "] = " << ax[e] << ";\n";
        }
      } else {
        for (int e = 0; e < NE; e++) o << "      v[" << e << "] = " << ax[e] << ";\n";
      }
      if (early && p == 0) o << "      }\n";
    }
    if (early && ld && p == last) o << "      " << GS << "\n      " << next_issue << "\n";
    // lazy zeros: a thread whose part of the tile index meets a still-zero
    // qubit holds only zeros in the first phase, which every op keeps zero
    const bool zskip_ops = sl.zfill_cap && p == 0;  // (zfill kernels never fold phase 0)
    if (zskip_ops) o << "      if (zt == 0u) {\n";
    for (int oi = P.op_begin; oi < P.op_end; oi++) {
      const ShmOp &op = ops[oi];
      const double *c = coef + op.coef;
      if (op.type == OP_DIAG) {
        // a run of consecutive factor-slot ops (one diagonal run): the
        // per-element factor is the product of the slots covering it;
        // unconditional slot factors are multiplied here (one literal per
        // element), conditional ones once per thread at run time and shared
        // between elements through partial products
        int oj = oi;
        while (oj < P.op_end && ops[oj].type == OP_DIAG) oj++;
        struct Slot {
          int sel;
          std::complex<double> lit;
          int rt;  // runtime factor index or -1
        };
        std::vector<Slot> slots;
        int nrt = 0;
        o << "      {\n";
        for (int q = oi; q < oj; q++) {
          const ShmOp &dq = ops[q];
          const double *cq = coef + dq.coef;
          const int eb = (int)dq.base_mask, ee = (int)dq.base_val;
          Slot sl_{kDiagSel[dq.t0], {cq[0], cq[1]}, -1};
          if (eb != ee) {
            sl_.rt = nrt++;
            // accumulated in R (fp32 runs: the product of a few unit phases
            // stays far inside BJ's 1e-4; keeps the 64-register budget)
            o << "        T fr" << sl_.rt << "; { R fx = " << lit(cq[0], f32) << ", fy = "
              << lit(cq[1], f32) << ";\n";
            const auto bit = bslot.find(q);
            if (bit != bslot.end())
              o << "          { const T bb = bfac[" << (pipe ? "(grp * 2 + itp) * " : "itp * ") << NB << " + "
                << bit->second << "]; const R nx = fx * bb.x - fy * bb.y; fy = fx * bb.y + fy * bb.x; fx = nx; }\n";
            const auto tit = tslot.find(q);
            if (tit != tslot.end())
              o << "          { const T tt = tfac[" << tit->second * NT
                << " + tid]; const R nx = fx * tt.x - fy * tt.y; fy = fx * tt.y + fy * tt.x; fx = nx; }\n";
            for (int i = eb; i < ee; i++) {
              const DiagEnt &d = ents[i];
              if (bit != bslot.end() && d.thr_mask == 0 && d.has_base) continue;
              if (tit != tslot.end() && d.thr_mask != 0 && !d.has_base) continue;
              o << "          if (((jt & " << d.thr_mask << ") == " << d.thr_val << ")";
              if (d.has_base)
                o << " && ((base & " << u64lit(d.base_mask) << ") == " << u64lit(d.base_val) << ")";
              o << ") { const R nx = fx * " << lit(d.re, f32) << " - fy * " << lit(d.im, f32)
                << "; fy = fx * " << lit(d.im, f32) << " + fy * " << lit(d.re, f32) << "; fx = nx; }\n";
            }
            o << "          fr" << sl_.rt << ".x = (R)fx; fr" << sl_.rt << ".y = (R)fy; }\n";
            sl_.lit = 1.0;
          }
          slots.push_back(sl_);
        }
        std::map<unsigned, std::string> prod;  // set of runtime factors -> variable
        int ng = 0;
        std::function<std::string(unsigned)> product = [&](unsigned set) -> std::string {
          auto it = prod.find(set);
          if (it != prod.end()) return it->second;
          const int hi = 31 - __builtin_clz(set);
          const unsigned rest = set & ~(1u << hi);
          std::string nm;
          if (!rest) {
            nm = "fr" + std::to_string(hi);
          } else {
            const std::string a = product(rest);
            nm = "g" + std::to_string(ng++);
            o << "        T " << nm << "; " << nm << ".x = " << a << ".x * fr" << hi << ".x - " << a
              << ".y * fr" << hi << ".y; " << nm << ".y = " << a << ".x * fr" << hi << ".y + " << a
              << ".y * fr" << hi << ".x;\n";
          }
          prod[set] = nm;
          return nm;
        };
        for (int e = 0; e < NE; e++) {
          std::complex<double> L = 1.0;
          unsigned rset = 0;
          for (auto &q : slots)
            if ((e & q.sel) == q.sel) {
              if (q.rt >= 0) rset |= 1u << q.rt;
              else L *= q.lit;
            }
          if (rset) {
            const std::string g = product(rset);
            o << "        { const T a = v[" << e << "]; v[" << e << "].x = " << g << ".x * a.x - " << g
              << ".y * a.y; v[" << e << "].y = " << g << ".x * a.y + " << g << ".y * a.x; }\n";
          }
          emit_cmul_lit(o, e, L.real(), L.imag(), f32, "        ");
        }
        o << "      }\n";
        oi = oj - 1;
        continue;
      }
      const bool full = (op.flags & OPF_FULL) != 0;
      const unsigned em = full ? 0xffffu : op.emask;
      const char *ind = "      ";
      if (!full) {
        o << "      if (";
        bool any = false;
        if (op.base_mask) {
          o << "((base & " << u64lit(op.base_mask) << ") == " << u64lit(op.base_val) << ")";
          any = true;
        }
        if (op.thr_mask) {
          if (any) o << " && ";
          o << "((jt & " << op.thr_mask << ") == " << op.thr_val << ")";
          any = true;
        }
        if (!any) o << "true";
        o << ") {\n";
        ind = "        ";
      }
      switch (op.type) {
        case OP_PHASE:
          for (int e = 0; e < NE; e++)
            if ((em >> e) & 1) emit_cmul_lit(o, e, c[0], c[1], f32, ind);
          break;
        case OP_DENSE1: {
          const int tb = op.t0;
          // an unconditional real block c * (+-1 entries) (H and its sign
          // variants): adds/subtracts only; the uniform factor c is deferred
          // (a scalar on every amplitude commutes with every op) and folded
          // into the next unconditional general block, else applied once
          // before the kernel's last store
          const bool sign_blk = full && defer_scalar && c[1] == 0 && c[3] == 0 && c[5] == 0 && c[7] == 0 &&
                                c[0] != 0 && std::abs(c[2]) == std::abs(c[0]) &&
                                std::abs(c[4]) == std::abs(c[0]) && std::abs(c[6]) == std::abs(c[0]);
          if (sign_blk) {
            const double k = std::abs(c[0]);
            pend *= k;
            const char *sg[4];
            for (int i = 0; i < 4; i++) sg[i] = c[2 * i] > 0 ? "+" : "-";
            for (int e = 0; e < NE; e++) {
              if (e & (1 << tb)) continue;
              const int e1 = e | (1 << tb);
              o << ind << "{ const T x0 = v[" << e << "], x1 = v[" << e1 << "];";
              for (int r = 0; r < 2; r++)
                for (int part = 0; part < 2; part++) {
                  const char *f = part ? "y" : "x";
                  o << " v[" << (r ? e1 : e) << "]." << f << " = " << sg[2 * r] << "x0." << f << " "
                    << sg[2 * r + 1] << " x1." << f << ";";
                }
              o << " }\n";
            }
            break;
          }
          // an unconditional real rotation [[a,-b],[b,a]] or reflection
          // [[a,b],[b,-a]]: factor out the larger of |a|, |b| (deferred like
          // the sign blocks), leaving one FMA per output component
          if (full && defer_scalar && c[1] == 0 && c[3] == 0 && c[5] == 0 && c[7] == 0) {
            const double a = c[0], b = c[4], m01 = c[2], m11 = c[6];
            const double tol = 1e-15 * (std::abs(a) + std::abs(b));
            const bool rot = std::abs(m11 - a) <= tol && std::abs(m01 + b) <= tol;
            const bool refl = std::abs(m11 + a) <= tol && std::abs(m01 - b) <= tol;
            if ((rot || refl) && a != 0 && b != 0) {
              const bool big_a = std::abs(a) >= std::abs(b);
              const double k = big_a ? a : b, t = big_a ? b / a : a / b;
              pend *= k;
              const std::string T_ = lit(t, f32), NT_ = lit(-t, f32);
              for (int e = 0; e < NE; e++) {
                if (e & (1 << tb)) continue;
                const int e1 = e | (1 << tb);
                o << ind << "{ const T x0 = v[" << e << "], x1 = v[" << e1 << "];";
                for (int part = 0; part < 2; part++) {
                  const char *f = part ? "y" : "x";
                  std::string y0, y1;
                  const std::string X0 = std::string("x0.") + f, X1 = std::string("x1.") + f;
                  if (rot && big_a) {        // (x0 - t x1, t x0 + x1)
                    y0 = "fma(" + NT_ + ", " + X1 + ", " + X0 + ")";
                    y1 = "fma(" + T_ + ", " + X0 + ", " + X1 + ")";
                  } else if (rot) {          // (t x0 - x1, x0 + t x1)
                    y0 = "fma(" + T_ + ", " + X0 + ", -" + X1 + ")";
                    y1 = "fma(" + T_ + ", " + X1 + ", " + X0 + ")";
                  } else if (big_a) {        // (x0 + t x1, t x0 - x1)
                    y0 = "fma(" + T_ + ", " + X1 + ", " + X0 + ")";
                    y1 = "fma(" + T_ + ", " + X0 + ", -" + X1 + ")";
                  } else {                   // (t x0 + x1, x0 - t x1)
                    y0 = "fma(" + T_ + ", " + X0 + ", " + X1 + ")";
                    y1 = "fma(" + NT_ + ", " + X1 + ", " + X0 + ")";
                  }
                  o << " v[" << e << "]." << f << " = " << y0 << "; v[" << e1 << "]." << f << " = " << y1 << ";";
                }
                o << " }\n";
              }
              break;
            }
          }
          // an unconditional [[a, ib], [ib, a]] (RX type): factor out the
          // larger of |a|, |b| likewise
          if (full && defer_scalar && c[1] == 0 && c[7] == 0 && c[2] == 0 && c[4] == 0 && c[0] == c[6] &&
              c[3] == c[5] && c[0] != 0 && c[3] != 0) {
            const double a = c[0], b = c[3];
            const bool big_a = std::abs(a) >= std::abs(b);
            const double k = big_a ? a : b, t = big_a ? b / a : a / b;
            pend *= k;
            const std::string T_ = lit(t, f32), NT_ = lit(-t, f32);
            for (int e = 0; e < NE; e++) {
              if (e & (1 << tb)) continue;
              const int e1 = e | (1 << tb);
              o << ind << "{ const T x0 = v[" << e << "], x1 = v[" << e1 << "];";
              if (big_a)  // y0 = x0 + i t x1, y1 = i t x0 + x1
                o << " v[" << e << "].x = fma(" << NT_ << ", x1.y, x0.x); v[" << e << "].y = fma(" << T_
                  << ", x1.x, x0.y); v[" << e1 << "].x = fma(" << NT_ << ", x0.y, x1.x); v[" << e1
                  << "].y = fma(" << T_ << ", x0.x, x1.y);";
              else  // y0 = t x0 + i x1, y1 = i x0 + t x1
                o << " v[" << e << "].x = fma(" << T_ << ", x0.x, -x1.y); v[" << e << "].y = fma(" << T_
                  << ", x0.y, x1.x); v[" << e1 << "].x = fma(" << T_ << ", x1.x, -x0.y); v[" << e1
                  << "].y = fma(" << T_ << ", x1.y, x0.x);";
              o << " }\n";
            }
            break;
          }
          double cs[8];
          for (int i = 0; i < 8; i++) cs[i] = c[i] * (full ? pend : 1.0);
          if (full) pend = 1.0;
          for (int e = 0; e < NE; e++) {
            if (e & (1 << tb)) continue;
            if (!((em >> e) & 1)) continue;
            const int idx[2] = {e, e | (1 << tb)};
            emit_block(o, 2, idx, cs, f32, ind);
          }
          break;
        }
        case OP_PERM1: {
          const int tb = op.t0;
          for (int e = 0; e < NE; e++) {
            if (e & (1 << tb)) continue;
            if (!((em >> e) & 1)) continue;
            o << ind << "{ const T a = v[" << e << "]; v[" << e << "] = v[" << (e | (1 << tb)) << "]; v["
              << (e | (1 << tb)) << "] = a; }\n";
          }
          break;
        }
        default: {  // OP_DENSE2
          const int t0 = op.t0, t1 = op.t1;
          for (int e = 0; e < NE; e++) {
            if (e & ((1 << t0) | (1 << t1))) continue;
            if (!((em >> e) & 1)) continue;
            const int idx[4] = {e, e | (1 << t0), e | (1 << t1), e | (1 << t0) | (1 << t1)};
            emit_block(o, 4, idx, c, f32, ind);
          }
        }
      }
      if (!full) o << "      }\n";
    }
    if (p == last && pend != 1.0) {
      for (int e = 0; e < NE; e++)
        o << "      v[" << e << "].x *= " << lit(pend, f32) << "; v[" << e << "].y *= " << lit(pend, f32) << ";\n";
      pend = 1.0;
    }
    if (zskip_ops) o << "      }\n";
    if (ld && p == last) {
      uint64_t limg[4] = {0, 0, 0, 0};
      for (int i = 0; i < RB; i++) limg[i] = sl.lcol[P.rbit[i]];
      o << "      u64 cg = gthr;\n";
      if (P.permuted) {
        o << "      cg ^= " << u64lit(PB(sl.lc0)) << ";\n";
        for (int i = P.term_begin; i < P.term_end; i++)
          o << "      if ((base & " << u64lit(terms[i].base_mask) << ") == " << u64lit(terms[i].base_val)
            << ") cg ^= " << u64lit(PB(terms[i].gvec)) << ";\n";
      }
      std::map<uint64_t, int> blk;
      if (pgp) {
        o << "      const u64 yb = obase | cg; const int bt = (int)(yb >> " << PSH << ");\n";
        for (int e = 0; e < NE; e++) {
          uint64_t x = 0;
          for (int i = 0; i < RB; i++)
            if ((e >> i) & 1) x ^= limg[i];
          const uint64_t c = PB(x) >> PSH;
          if (!blk.count(c)) {
            const int k = (int)blk.size();
            blk[c] = k;
            o << "      T *pd" << k << " = ptab_s[bt ^ " << c << "]; __builtin_assume(__isGlobal(pd" << k << "));\n";
          }
        }
      }
      for (int e = 0; e < NE; e++) {
        uint64_t x = 0;
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) x ^= limg[i];
        if (pgp)
          o << "      pd" << blk[PB(x) >> PSH] << "[(yb ^ " << u64lit(PB(x)) << ") & " << u64lit((1ull << PSH) - 1)
            << "] = v[" << e << "];\n";
        else
          o << "      " << (operm ? "dst[obase" : "st[base") << " | (cg ^ " << u64lit(PB(x)) << ")] = v[" << e << "];\n";
      }
      o << "    }\n";
      break;
    }
    if (P.permuted) {
      o << "      u32 cb = " << Sx(swzs[ssw[p]], Ac0[p]) << "u;\n";
      for (int i = P.term_begin; i < P.term_end; i++)
        o << "      if ((base & " << u64lit(terms[i].base_mask) << ") == " << u64lit(terms[i].base_val)
          << ") cb ^= " << Sx(swzs[ssw[p]], Sx(GL, terms[i].vec_swz)) << "u;\n";
      o << "      const int s0 = (int)(stab[" << sslot[p] * NT << " + tid] ^ cb);\n";
      o << "      " << GS << "\n";
      for (int e = 0; e < NE; e++) {
        int a = 0;
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) a ^= simg[p][P.rbit[i]];
        o << "      tb[s0 ^ " << a << "] = v[" << e << "];\n";
      }
    } else {
      std::vector<int> as(NE, 0);
      for (int e = 0; e < NE; e++)
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) as[e] ^= sr[i];
      const auto ax = addr_group("sj", as, "      ");
      for (int e = 0; e < NE; e++) o << "      " << ax[e] << " = v[" << e << "];\n";
    }
    o << "      " << GS << "\n    }\n";
  }
  if (!ld) {
    std::map<uint64_t, int> oblk;
    if (pgp) {
      o << "    { const u64 gy = obase + ooff_t;\n";
      for (int it = 0; it < NE; it++) {
        const uint64_t c = PB(itoff[it]) >> PSH;
        if (!oblk.count(c)) {
          const int k = (int)oblk.size();
          oblk[c] = k;
          o << "      T *od" << k << " = ptab_s[(int)(gy >> " << PSH << ") | " << c << "] + (gy & "
            << u64lit((1ull << PSH) - 1) << "); __builtin_assume(__isGlobal(od" << k << "));\n";
        }
      }
    } else {
      o << (operm ? "    { T *g = dst + obase + ooff_t;\n" : "    { T *g = st + base + off_t;\n");
    }
    auto gst = [&](int it) {
      return pgp ? "od" + std::to_string(oblk[PB(itoff[it]) >> PSH]) + "[" +
                       u64lit(PB(itoff[it]) & ((1ull << PSH) - 1)) + "]"
                 : "g[" + u64lit(PB(itoff[it])) + "]";
    };
    if (early) {
      std::vector<int> as;
      for (int it = 0; it < NE; it++) as.push_back((int)Sx(SO, (unsigned)(it * NT)));
      const auto ax = addr_group("sw_out", as, "      ");
      for (int it = 0; it < NE; it++) o << "      v[" << it << "] = " << ax[it] << ";\n";
      o << "      " << GS << "\n      " << next_issue << "\n";
      for (int it = 0; it < NE; it++) o << "      " << gst(it) << " = v[" << it << "];\n";
    } else {
      std::vector<int> as;
      for (int it = 0; it < NE; it++) as.push_back((int)Sx(SO, (unsigned)(it * NT)));
      const auto ax = addr_group("sw_out", as, "      ");
      for (int it = 0; it < NE; it++) o << "      " << gst(it) << " = " << ax[it] << ";\n";
    }
    o << "    }\n";
  }
  if (!early) o << "    __syncthreads();\n";
  if (!pipe) o << "    b = (b + 1) % " << nbuf << ";\n";
  if (NB) o << "    itp ^= 1;\n";
  o << "  }\n}\n";
  return o.str();
}

static bool shm_jit_zero_ok_src(const std::string &src) {
  return strstr(src.c_str(), "#define ZERO_OK 1") != nullptr;
}

size_t shm_jit_smem(const std::string &src) {
  const char *p = strstr(src.c_str(), "#define SMEM_BYTES ");
  return p ? (size_t)strtoull(p + 19, nullptr, 10) : 0;
}

// Compile (NVRTC, sm_100a) every source not yet in the process cache; the
// distinct sources are spread over host threads.
static std::vector<JitEntry *> jit_compile_all(const std::vector<std::string> &srcs,
                                               const std::vector<std::string> &names) {
  nvrtc_load();
  std::vector<JitEntry *> out(srcs.size(), nullptr);
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t i = 0; i < srcs.size(); i++) {
      auto it = g_cache.find(srcs[i]);
      if (it != g_cache.end()) out[i] = it->second;
      else todo.push_back(i);
    }
  }
  std::vector<std::string> errs(srcs.size());
  std::vector<std::vector<char>> cubins(srcs.size());
  std::atomic<size_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const size_t w = next.fetch_add(1);
      if (w >= todo.size()) return;
      const size_t i = todo[w];
      nvrtcProgram_ prog = nullptr;
      int r = g_nvrtc.create(&prog, srcs[i].c_str(), (names[i] + ".cu").c_str(), 0, nullptr, nullptr);
      if (r != 0) {
        errs[i] = std::string("nvrtcCreateProgram: ") + g_nvrtc.err(r);
        continue;
      }
      const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-default-device"};
      r = g_nvrtc.compile(prog, 4, opts);
      if (r != 0) {
        size_t ls = 0;
        g_nvrtc.logSize(prog, &ls);
        std::string log(ls, '\0');
        g_nvrtc.log(prog, &log[0]);
        errs[i] = std::string("nvrtcCompileProgram: ") + g_nvrtc.err(r) + "\n" + log.substr(0, 2000);
        g_nvrtc.destroy(&prog);
        continue;
      }
      size_t cs = 0;
      g_nvrtc.cubinSize(prog, &cs);
      cubins[i].resize(cs);
      g_nvrtc.cubin(prog, cubins[i].data());
      g_nvrtc.destroy(&prog);
    }
  };
  unsigned nth = std::thread::hardware_concurrency();
  if (nth == 0) nth = 4;
  nth = std::min<unsigned>(nth, 32);
  nth = std::min<unsigned>(nth, (unsigned)std::max<size_t>(todo.size(), 1));
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nth; t++) th.emplace_back(worker);
  worker();
  for (auto &t : th) t.join();
  for (size_t i : todo)
    if (!errs[i].empty()) fail(ATLAS_E_CUDA, "shm_jit: %s", errs[i].c_str());
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (size_t i : todo) {
    auto it = g_cache.find(srcs[i]);
    if (it != g_cache.end()) {  // same source twice in this batch
      out[i] = it->second;
      continue;
    }
    JitEntry *E = new JitEntry();
    cudaError_t e = cudaLibraryLoadData(&E->lib, cubins[i].data(), nullptr, nullptr, 0, nullptr,
                                        nullptr, 0);
    if (e != cudaSuccess) fail(ATLAS_E_CUDA, "cudaLibraryLoadData: %s", cudaGetErrorString(e));
    e = cudaLibraryGetKernel(&E->kern, E->lib, names[i].c_str());
    if (e != cudaSuccess) fail(ATLAS_E_CUDA, "cudaLibraryGetKernel: %s", cudaGetErrorString(e));
    E->smem = (int)shm_jit_smem(srcs[i]);
    if (const char *tp = strstr(srcs[i].c_str(), "#define ATLAS_TMA ")) {
      tp += 18;
      E->tma_rank = (int)strtol(tp, (char **)&tp, 10);
      for (int d = 0; d < E->tma_rank; d++) {
        E->tstart[d] = (int)strtol(tp, (char **)&tp, 10);
        E->tlen[d] = (int)strtol(tp + 1, (char **)&tp, 10);
        E->tabits[d] = (int)strtol(tp + 1, (char **)&tp, 10);
      }
    }
    E->zero_ok = shm_jit_zero_ok_src(srcs[i]);
    {
      const char *p = strstr(srcs[i].c_str(), "#define BLOCK_THREADS ");
      E->threads = p ? atoi(p + 22) : 0;
    }
    g_cache[srcs[i]] = E;
    out[i] = E;
  }
  return out;
}

// Generate and compile the specialised kernel of every L_SHM launch of the
// plan (all simulated ranks); Launch::jit points at the cache entry.
// Lazy-zero chains (runtime.cu): the stage-0 launches after the first, up to
// the one that makes every local slot active, carry the zero-fill load; the
// chain holds only if every launch in it is an in-place shared-memory launch.
void shm_mark_zfill(atlas_ctx *C) {
  const uint64_t lmask = C->L >= 64 ? ~0ull : (1ull << C->L) - 1;
  for (auto &P : C->prog) {
    for (auto &ln : P) ln.sl.zfill_cap = 0;
    if (!C->opt.zero_skip || !C->opt.zero_lazy || C->opt.shm_tma || !C->opt.shm_jit) continue;
    uint64_t z = lmask;
    bool ok = false;
    size_t i = 0;
    for (; i < P.size() && P[i].stage == 0; i++) {
      if (P[i].type != L_SHM || P[i].sl.out_perm_off >= 0) break;
      z &= P[i].sl.nonactive;
      if (!z) {
        ok = true;
        break;
      }
    }
    if (ok)
      for (size_t j = 1; j <= i; j++) P[j].sl.zfill_cap = 1;
  }
}

// Autotuning (option shm_autotune): every shared-memory launch gets up to
// four variants compiled -- tile pipeline (one CTA of two thread groups on a
// ring of three buffers, or two single-buffer CTAs per SM) x last phase
// stored straight to HBM or copied out through shared memory; runtime.cu
// times each once in the first runs after the plan and keeps the fastest per
// launch (measured per-launch differences of up to 13% either way, not
// predictable from the phase count).
void shm_jit_prepare(atlas_ctx *C) {
  std::vector<std::string> srcs, names;
  std::vector<std::pair<Launch *, int>> lns;  // (launch, variant index)
  auto add = [&](Launch *ln, int force_pipe, int force_ld) {
    g_force_pipe = force_pipe;
    g_force_ld = force_ld;
    std::string body;
    try {
      body = shm_jit_source(C, ln->sl, "atlas_shm_jit");
    } catch (...) {
      g_force_pipe = -1;
      g_force_ld = -1;
      throw;
    }
    g_force_pipe = -1;
    g_force_ld = -1;
    // the name does not enter the cache key: it is derived from the body
    const size_t h = std::hash<std::string>()(body);
    char nm[64];
    snprintf(nm, sizeof nm, "atlas_shm_%016zx", h);
    std::string s = body;
    const size_t at = s.find("atlas_shm_jit");
    s.replace(at, strlen("atlas_shm_jit"), nm);
    for (size_t i = 0; i < srcs.size(); i++)
      if (lns[i].first == ln && srcs[i] == s) return;  // the same kernel as a variant already listed
    srcs.push_back(s);
    names.push_back(nm);
    lns.push_back({ln, ln->nvar++});
  };
  shm_mark_zfill(C);
  for (auto &P : C->prog)
    for (auto &ln : P)
      if (ln.type == L_SHM) {
        ln.nvar = 0;
        ln.tune_warm = false;
        for (int v = 0; v < 4; v++) {
          ln.jit_var[v] = nullptr;
          ln.tune_ms[v] = -1.f;
        }
        add(&ln, -1, -1);
        if (C->opt.shm_autotune) {
          // (fp32 tiles never use the two-group pipeline: the pipeline
          // variants then generate the same source and are dropped)
          if (C->opt.shm_pipe) add(&ln, 0, -1);
          if (ln.sl.last_direct) {
            add(&ln, -1, 0);
            if (C->opt.shm_pipe) add(&ln, 0, 0);
          }
        }
      }
  if (srcs.empty()) return;
  auto ents = jit_compile_all(srcs, names);
  for (size_t i = 0; i < lns.size(); i++) lns[i].first->jit_var[lns[i].second] = ents[i];
  for (auto &P : C->prog)
    for (auto &ln : P)
      if (ln.type == L_SHM) {
        ln.jit = ln.jit_var[0];
        if (ln.nvar < 2) ln.nvar = 0;  // nothing to tune
      }
  // load every kernel now (dynamic shared-memory limit, occupancy): a
  // first launch that loads its module stalls the stream and would count
  // against its variant in the tuning runs
  for (size_t i = 0; i < ents.size(); i++) shm_jit_prime(ents[i]);
}

static int g_nsms = 0;
static std::mutex g_tmap_mu;

bool shm_jit_zero_ok(const void *jit) { return jit && ((const JitEntry *)jit)->zero_ok; }

// Set the kernel's dynamic shared-memory limit and read its occupancy (once
// per kernel; this also loads the module).
static cudaError_t jit_prime(JitEntry *E, int NT) {
  if (E->attr_set >= E->smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute((const void *)E->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, E->smem);
  if (e != cudaSuccess) return e;
  E->attr_set = E->smem;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)E->kern, NT, E->smem);
  if (e != cudaSuccess) return e;
  E->nt = occ < 1 ? 1 : occ;
  return cudaSuccess;
}
void shm_jit_prime(void *jit) {
  JitEntry *E = (JitEntry *)jit;
  if (E && E->threads > 0) {
    cudaError_t e = jit_prime(E, E->threads);
    if (e != cudaSuccess) fail(ATLAS_E_CUDA, "shm_jit prime: %s", cudaGetErrorString(e));
  }
}

// skip: non-active slots whose tiles with a 1 there are zero in and out (the
// launch runs in place); those tiles are not visited at all
cudaError_t launch_shm_jit(void *jit, void *st, void *dst, const ShmLaunch &sl, cudaStream_t s, int zmode,
                           uint64_t skip, void *const *peers, uint64_t zq) {
  JitEntry *E = (JitEntry *)jit;
  const int NT = E->threads > 0 ? E->threads : 1 << (sl.K - sl.RB);
  {
    cudaError_t e = jit_prime(E, NT);
    if (e != cudaSuccess) return e;
  }
  if (!g_nsms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsms, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsms <= 0) g_nsms = 148;
  }
  // TMA: the shard (the launch reads st) as a <= 5-dimensional fp64 tensor
  // whose dimensions are the runs of local slots of the generated kernel
  // (tma_dims); the box is the tile, 128-B swizzled
  void *tmg = nullptr;
  if (E->tma_rank) {
    std::lock_guard<std::mutex> lk(g_tmap_mu);
    auto it = E->dmaps.find(st);
    if (it != E->dmaps.end()) tmg = it->second;
  }
  if (E->tma_rank && !tmg) {
    alignas(64) CUtensorMap tmap;
    typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);
    static EncodeTiled enc = nullptr;
    if (!enc) {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
      if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
      enc = (EncodeTiled)fn;
    }
    cuuint64_t gdim[5], gstr[4];
    cuuint32_t box[5], es[5];
    for (int d = 0; d < E->tma_rank; d++) {
      gdim[d] = d == 0 ? 16 : (cuuint64_t)1 << E->tlen[d];
      box[d] = d == 0 ? 16 : 1u << E->tabits[d];
      es[d] = 1;
      if (d > 0) gstr[d - 1] = (cuuint64_t)16 << E->tstart[d];
    }
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)E->tma_rank, st, gdim, gstr, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    cudaError_t e = cudaMalloc(&tmg, sizeof(CUtensorMap));
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(tmg, &tmap, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_tmap_mu);
    E->dmaps[st] = tmg;
  }
  uint64_t nact = sl.nonactive & ~skip;
  uint32_t ntl = (uint32_t)(sl.ntiles >> __builtin_popcountll(sl.nonactive & skip));
  uint64_t grid = (uint64_t)g_nsms * E->nt;
  if (grid > ntl) grid = ntl;
  if (sl.grid_cap > 0 && grid > (uint64_t)sl.grid_cap) grid = (uint64_t)sl.grid_cap;
  struct PeerTab {
    void *p[8];
  } ptab = {};
  if (sl.peer_gp > 0) {
    if (!peers) return cudaErrorInvalidValue;
    for (int b = 0; b < (1 << sl.peer_gp); b++) ptab.p[b] = peers[b];
  }
  // zq: local slots still |0> with lazy zeros -> the active ones as tile bits
  uint32_t zfill = 0;
  for (int b = 0; b < sl.K; b++)
    if ((zq >> sl.act[b]) & 1) zfill |= 1u << b;
  void *args[8] = {&st, &dst, &zmode, &nact, &ntl, &zfill};
  int na = 6;
  if (E->tma_rank) args[na++] = &tmg;
  if (sl.peer_gp > 0) args[na++] = &ptab;
  return cudaLaunchKernel((const void *)E->kern, dim3((unsigned)grid), dim3(NT), args,
                          (size_t)E->smem, s);
}

// source of launch i of slot s (tests / inspection: atlas_get_jit_source)
std::string shm_jit_source_of(const atlas_ctx *C, int slot, int i) {
  if (slot < 0 || slot >= (int)C->prog.size()) fail(ATLAS_E_INVALID, "slot out of range");
  shm_mark_zfill(const_cast<atlas_ctx *>(C));  // the same flags the run compiles with
  int j = 0;
  for (auto &ln : C->prog[slot])
    if (ln.type == L_SHM && j++ == i) return shm_jit_source(C, ln.sl, "atlas_shm_jit");
  fail(ATLAS_E_INVALID, "no shared-memory launch %d", i);
  return "";
}

}  // namespace atlas
