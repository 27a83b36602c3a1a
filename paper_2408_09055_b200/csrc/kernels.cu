// kernels.cu -- sm_100a device kernels of the Atlas hot path.
//
//  fused_kernel   PAPER.md P:L1962 "Fusion": apply one 2^k x 2^k matrix to
//                 every group of 2^k amplitudes whose indices differ only in
//                 the k target bits (Eq. 2 generalised).
//  shm_kernel     P:L1964 "Shared-memory": stage a 2^K-amplitude tile of the
//                 active qubits in shared memory and apply the kernel's gates
//                 one by one (register phases, insular selectors on any local
//                 qubit).
//  permute_kernel the local bit permutation of the inter-stage remap (Alg.
//                 Execute's Shard).
//  scale_kernel   per-rank scalar of insular gates on global qubits when a
//                 stage has no kernel to fold it into.
//
// Every kernel is HBM-streaming: each launch reads and writes every amplitude
// of the shard exactly once (2 * 2^L * sizeof(amp) algorithmic bytes).
#include <utility>
#include <cuda_runtime.h>

#include <cstdint>

#include "device.h"

namespace atlas {

template <typename R> struct Cplx;
template <> struct Cplx<double> { using T = double2; };
template <> struct Cplx<float> { using T = float2; };

// ------------------------------------------------------------------ helpers
__host__ __device__ constexpr int ctz_c(int e) { return (e & 1) ? 0 : 1 + ctz_c(e >> 1); }

__device__ __forceinline__ uint64_t pdep64(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  while (mask) {
    uint64_t lo = mask & (~mask + 1);
    if (v & 1) r |= lo;
    v >>= 1;
    mask ^= lo;
  }
  return r;
}

template <typename R> __host__ __device__ constexpr int swz(int j);
template <> __host__ __device__ constexpr int swz<double>(int j) { return swz_c128(j); }
template <> __host__ __device__ constexpr int swz<float>(int j) { return swz_c64(j); }

template <typename T>
__device__ __forceinline__ void cmac(T &acc, const T &a, const T &x) {
  acc.x = fma(a.x, x.x, acc.x);
  acc.x = fma(-a.y, x.y, acc.x);
  acc.y = fma(a.x, x.y, acc.y);
  acc.y = fma(a.y, x.x, acc.y);
}

template <typename T>
__device__ __forceinline__ T cmul(const T &a, const T &x) {
  T r;
  r.x = a.x * x.x - a.y * x.y;
  r.y = a.x * x.y + a.y * x.x;
  return r;
}

template <typename T>
__device__ __forceinline__ void cp_async(T *smem, const T *gmem);
template <>
__device__ __forceinline__ void cp_async<double2>(double2 *smem, const double2 *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <>
__device__ __forceinline__ void cp_async<float2>(float2 *smem, const float2 *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ------------------------------------------------------------ fused kernel
template <typename R, int k>
__global__ void __launch_bounds__(256) fused_kernel(typename Cplx<R>::T *__restrict__ st,
                                                    uint64_t ngroups, FusedLaunch fl,
                                                    const double2 *__restrict__ mats) {
  using T = typename Cplx<R>::T;
  constexpr int D = 1 << k;
  extern __shared__ unsigned char smraw[];
  T *M = reinterpret_cast<T *>(smraw);
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) {
    double2 m = mats[fl.mat_off + i];
    M[i].x = (R)m.x;
    M[i].y = (R)m.y;
  }
  __syncthreads();
  uint64_t bit[k];
#pragma unroll
  for (int j = 0; j < k; j++) bit[j] = 1ull << fl.t[j];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += stride) {
    // base = g with zero bits inserted at the (ascending) target slots:
    // f(i) of Eq. 2 applied once per target.
    uint64_t base = g;
#pragma unroll
    for (int j = 0; j < k; j++) {
      const uint64_t lo = base & (bit[j] - 1);
      base = ((base ^ lo) << 1) | lo;
    }
    T x[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
      uint64_t off = 0;
#pragma unroll
      for (int j = 0; j < k; j++)
        if ((c >> j) & 1) off |= bit[j];
      x[c] = st[base + off];
    }
    // rows are produced one at a time (x stays in registers; the row loop is
    // not unrolled so only one accumulator is live)
#pragma unroll 1
    for (int r = 0; r < D; r++) {
      T acc;
      acc.x = 0;
      acc.y = 0;
      const T *Mr = M + r * D;
#pragma unroll
      for (int c = 0; c < D; c++) cmac(acc, Mr[c], x[c]);
      uint64_t off = 0;
#pragma unroll
      for (int j = 0; j < k; j++)
        if ((r >> j) & 1) off |= bit[j];
      st[base + off] = acc;
    }
  }
}

// ------------------------------------------------------------- shm kernel
// Register-element loops are fully unrolled: e (and the pair partner) are
// compile-time.  CHK = the op is conditional: it applies where the runtime
// element mask has bit e set and the thread predicate `ok` holds; unconditional
// ops (OPF_FULL) compile to straight-line code.
template <typename T, int NE, int TB, bool CHK>
__device__ __forceinline__ void dense1(T (&v)[NE], const T (&m)[4], unsigned emask, bool ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & (1 << TB)) continue;
    const int e1 = e | (1 << TB);
    if (!CHK || (ok && ((emask >> e) & 1u))) {
      const T a = v[e], b = v[e1];
      T y0, y1;
      y0.x = m[0].x * a.x;
      y0.y = m[0].x * a.y;
      y1.x = m[2].x * a.x;
      y1.y = m[2].x * a.y;
      y0.x = fma(-m[0].y, a.y, y0.x);
      y0.y = fma(m[0].y, a.x, y0.y);
      y1.x = fma(-m[2].y, a.y, y1.x);
      y1.y = fma(m[2].y, a.x, y1.y);
      cmac(y0, m[1], b);
      cmac(y1, m[3], b);
      v[e] = y0;
      v[e1] = y1;
    }
  }
}

// real 2x2 block (m[i].y == 0): 8 flops per pair instead of 16
template <typename T, int NE, int TB, bool CHK>
__device__ __forceinline__ void dense1r(T (&v)[NE], const T (&m)[4], unsigned emask, bool ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & (1 << TB)) continue;
    const int e1 = e | (1 << TB);
    if (!CHK || (ok && ((emask >> e) & 1u))) {
      const T a = v[e], b = v[e1];
      T y0, y1;
      y0.x = fma(m[1].x, b.x, m[0].x * a.x);
      y0.y = fma(m[1].x, b.y, m[0].x * a.y);
      y1.x = fma(m[3].x, b.x, m[2].x * a.x);
      y1.y = fma(m[3].x, b.y, m[2].x * a.y);
      v[e] = y0;
      v[e1] = y1;
    }
  }
}

template <typename T, int NE, int TB, bool CHK>
__device__ __forceinline__ void perm1(T (&v)[NE], unsigned emask, bool ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & (1 << TB)) continue;
    const int e1 = e | (1 << TB);
    if (!CHK || (ok && ((emask >> e) & 1u))) {
      const T a = v[e];
      v[e] = v[e1];
      v[e1] = a;
    }
  }
}

template <typename T, int NE, int TB0, int TB1, bool CHK>
__device__ __forceinline__ void dense2(T (&v)[NE], const double *__restrict__ m, unsigned emask,
                                       bool ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & ((1 << TB0) | (1 << TB1))) continue;
    if (!CHK || (ok && ((emask >> e) & 1u))) {
      const int idx[4] = {e, e | (1 << TB0), e | (1 << TB1), e | (1 << TB0) | (1 << TB1)};
      T x[4], y[4];
#pragma unroll
      for (int c = 0; c < 4; c++) x[c] = v[idx[c]];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        y[r].x = 0;
        y[r].y = 0;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          T a;
          a.x = m[2 * (r * 4 + c)];
          a.y = m[2 * (r * 4 + c) + 1];
          cmac(y[r], a, x[c]);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; r++) v[idx[r]] = y[r];
    }
  }
}

// multiply the elements selected by a factor slot (OP_DIAG) by f
template <typename T, int NE, int SEL>
__device__ __forceinline__ void diag_mul(T (&v)[NE], const T &f) {
#pragma unroll
  for (int e = 0; e < NE; e++)
    if ((e & SEL) == SEL) v[e] = cmul(f, v[e]);
}

template <typename R, int RB, bool CHK>
__device__ __forceinline__ void apply_op(typename Cplx<R>::T (&v)[1 << RB], const ShmOp &o,
                                         const double *__restrict__ coef, bool ok) {
  using T = typename Cplx<R>::T;
  constexpr int NE = 1 << RB;
  const unsigned em = o.emask;
  switch (o.type) {
    case OP_PHASE: {
      T c;
      c.x = (R)coef[o.coef];
      c.y = (R)coef[o.coef + 1];
#pragma unroll
      for (int e = 0; e < NE; e++)
        if (!CHK || (ok && ((em >> e) & 1u))) v[e] = cmul(c, v[e]);
      break;
    }
    case OP_DENSE1: {
      T m[4];
      // complex coefficients are 16-byte aligned pairs: one LDS.128 each
      const double2 *c2 = reinterpret_cast<const double2 *>(coef + o.coef);
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const double2 cc = c2[i];
        m[i].x = (R)cc.x;
        m[i].y = (R)cc.y;
      }
      if (!CHK && (o.flags & OPF_REAL)) {
        switch (o.t0) {
          case 0: dense1r<T, NE, 0, CHK>(v, m, em, ok); break;
          case 1: if (RB > 1) dense1r<T, NE, (RB > 1 ? 1 : 0), CHK>(v, m, em, ok); break;
          case 2: if (RB > 2) dense1r<T, NE, (RB > 2 ? 2 : 0), CHK>(v, m, em, ok); break;
          case 3: if (RB > 3) dense1r<T, NE, (RB > 3 ? 3 : 0), CHK>(v, m, em, ok); break;
        }
      } else {
        switch (o.t0) {
          case 0: dense1<T, NE, 0, CHK>(v, m, em, ok); break;
          case 1: if (RB > 1) dense1<T, NE, (RB > 1 ? 1 : 0), CHK>(v, m, em, ok); break;
          case 2: if (RB > 2) dense1<T, NE, (RB > 2 ? 2 : 0), CHK>(v, m, em, ok); break;
          case 3: if (RB > 3) dense1<T, NE, (RB > 3 ? 3 : 0), CHK>(v, m, em, ok); break;
        }
      }
      break;
    }
    case OP_PERM1:
      switch (o.t0) {
        case 0: perm1<T, NE, 0, CHK>(v, em, ok); break;
        case 1: if (RB > 1) perm1<T, NE, (RB > 1 ? 1 : 0), CHK>(v, em, ok); break;
        case 2: if (RB > 2) perm1<T, NE, (RB > 2 ? 2 : 0), CHK>(v, em, ok); break;
        case 3: if (RB > 3) perm1<T, NE, (RB > 3 ? 3 : 0), CHK>(v, em, ok); break;
      }
      break;
    default: {  // OP_DENSE2, t0 < t1
      const double *m = coef + o.coef;
      switch (o.t0 * 4 + o.t1) {
        case 1: if (RB > 1) dense2<T, NE, 0, (RB > 1 ? 1 : 0), CHK>(v, m, em, ok); break;
        case 2: if (RB > 2) dense2<T, NE, 0, (RB > 2 ? 2 : 0), CHK>(v, m, em, ok); break;
        case 3: if (RB > 3) dense2<T, NE, 0, (RB > 3 ? 3 : 0), CHK>(v, m, em, ok); break;
        case 6: if (RB > 2) dense2<T, NE, (RB > 2 ? 1 : 0), (RB > 2 ? 2 : 0), CHK>(v, m, em, ok); break;
        case 7: if (RB > 3) dense2<T, NE, (RB > 3 ? 1 : 0), (RB > 3 ? 3 : 0), CHK>(v, m, em, ok); break;
        case 11: if (RB > 3) dense2<T, NE, (RB > 3 ? 2 : 0), (RB > 3 ? 3 : 0), CHK>(v, m, em, ok); break;
      }
    }
  }
}

// OP_DIAG: accumulate the slot's factor (unconditional part times every
// conditional entry whose thread/tile condition holds), then multiply it in.
template <typename R, int RB>
__device__ __forceinline__ void apply_diag(typename Cplx<R>::T (&v)[1 << RB], const ShmOp &o,
                                           const double *__restrict__ coef,
                                           const DiagEnt *__restrict__ ents, int jt,
                                           uint64_t base) {
  using T = typename Cplx<R>::T;
  constexpr int NE = 1 << RB;
  // the factor is accumulated in fp64 (a product of many unit phases)
  double fx = coef[o.coef], fy = coef[o.coef + 1];
  const int eb = (int)o.base_mask, ee = (int)o.base_val;
  for (int i = eb; i < ee; i++) {
    const DiagEnt &d = ents[i];
    bool c = (jt & d.thr_mask) == d.thr_val;
    if (d.has_base) c = c && ((base & d.base_mask) == d.base_val);
    if (c) {
      const double nx = fx * d.re - fy * d.im;
      fy = fx * d.im + fy * d.re;
      fx = nx;
    }
  }
  T f;
  f.x = (R)fx;
  f.y = (R)fy;
  switch (o.t0) {
    case 0: diag_mul<T, NE, 0>(v, f); break;
    case 1: diag_mul<T, NE, 1>(v, f); break;
    case 2: if (RB > 1) diag_mul<T, NE, (RB > 1 ? 2 : 0)>(v, f); break;
    case 3: if (RB > 2) diag_mul<T, NE, (RB > 2 ? 4 : 0)>(v, f); break;
    case 4: if (RB > 3) diag_mul<T, NE, (RB > 3 ? 8 : 0)>(v, f); break;
    case 5: if (RB > 1) diag_mul<T, NE, (RB > 1 ? 3 : 0)>(v, f); break;
    case 6: if (RB > 2) diag_mul<T, NE, (RB > 2 ? 5 : 0)>(v, f); break;
    case 7: if (RB > 3) diag_mul<T, NE, (RB > 3 ? 9 : 0)>(v, f); break;
    case 8: if (RB > 2) diag_mul<T, NE, (RB > 2 ? 6 : 0)>(v, f); break;
    case 9: if (RB > 3) diag_mul<T, NE, (RB > 3 ? 10 : 0)>(v, f); break;
    case 10: if (RB > 3) diag_mul<T, NE, (RB > 3 ? 12 : 0)>(v, f); break;
  }
}

__host__ __device__ inline size_t shm_align16(size_t x) { return (x + 15) & ~(size_t)15; }

// dynamic shared memory layout of one launch (host and device agree)
struct ShmSmem {
  size_t ops, coef, phase, ents, terms, jtab, stab, itoff, btab, total;
};
__host__ __device__ inline ShmSmem shm_smem_layout(int tile_bytes, int nbuf, const ShmLaunch &sl,
                                                   int nt, int ne) {
  ShmSmem L;
  size_t o = (size_t)tile_bytes * nbuf;
  L.ops = o;
  o = shm_align16(o + (size_t)sl.nops * sizeof(ShmOp));
  L.coef = o;
  o = shm_align16(o + (size_t)sl.ncoef * sizeof(double));
  L.phase = o;
  o = shm_align16(o + (size_t)sl.nphase * sizeof(ShmPhase));
  L.ents = o;
  o = shm_align16(o + (size_t)sl.nent * sizeof(DiagEnt));
  L.terms = o;
  o = shm_align16(o + (size_t)sl.nterm * sizeof(PermTerm));
  L.jtab = o;
  o = shm_align16(o + (size_t)sl.nphase * nt * sizeof(uint32_t));
  L.stab = o;
  o = shm_align16(o + (size_t)sl.nphase * nt * sizeof(uint16_t));
  L.itoff = o;
  o = shm_align16(o + (size_t)ne * sizeof(uint64_t));
  L.btab = o;
  o = shm_align16(o + (size_t)4 * 256 * sizeof(uint64_t));
  L.total = o;
  return L;
}

// Persistent shared-memory kernel.  One CTA loops over tiles; with NBUF = 2
// the next tile's HBM->SMEM copy (cp.async) overlaps the current tile's
// register phases and store.  Everything that does not depend on the tile --
// the op program, per-phase thread indices and store offsets, per-iteration
// global offsets and the tile-base deposit tables -- is staged in SMEM once
// per CTA.  The swizzle is linear over GF(2), so shared addresses are XORs of
// per-thread and per-element parts; the same holds for the permuted store of
// a phase whose affine permutation gates were folded into its addresses.
// two CTAs per SM for the 256-thread configurations (register cap 128)
template <typename R, int K, int RB, int NBUF>
struct ShmMinBlocks {
  static constexpr int value = (NBUF == 1 && (K - RB) >= 8 && (K - RB) <= 9 && (sizeof(R) << (K + 1)) <= 65536) ? 2 : 1;
};

template <typename R, int K, int RB, int NBUF>
__global__ void __launch_bounds__(1 << (K - RB), (ShmMinBlocks<R, K, RB, NBUF>::value)) shm_kernel(
    typename Cplx<R>::T *__restrict__ st, ShmLaunch sl, const ShmOp *__restrict__ gops,
    const double *__restrict__ gcoef, const ShmPhase *__restrict__ gph,
    const DiagEnt *__restrict__ gents, const PermTerm *__restrict__ gterms) {
  using T = typename Cplx<R>::T;
  constexpr int NT = 1 << (K - RB);
  constexpr int NE = 1 << RB;
  constexpr int TILE = 1 << K;
  extern __shared__ __align__(16) unsigned char smraw[];
  const ShmSmem lay = shm_smem_layout(TILE * (int)sizeof(T), NBUF, sl, NT, NE);
  T *buf = reinterpret_cast<T *>(smraw);
  ShmOp *ops = reinterpret_cast<ShmOp *>(smraw + lay.ops);
  double *coef = reinterpret_cast<double *>(smraw + lay.coef);
  ShmPhase *ph = reinterpret_cast<ShmPhase *>(smraw + lay.phase);
  DiagEnt *ents = reinterpret_cast<DiagEnt *>(smraw + lay.ents);
  PermTerm *terms = reinterpret_cast<PermTerm *>(smraw + lay.terms);
  uint32_t *jtab = reinterpret_cast<uint32_t *>(smraw + lay.jtab);  // (swz(jt) << 16) | jt
  uint16_t *stab = reinterpret_cast<uint16_t *>(smraw + lay.stab);  // swz(A jt)
  uint64_t *itoff = reinterpret_cast<uint64_t *>(smraw + lay.itoff);
  uint64_t *btab = reinterpret_cast<uint64_t *>(smraw + lay.btab);
  const int tid = threadIdx.x;

  // ---- stage the program and the index tables
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(gops + sl.ops_off);
    uint4 *dst = reinterpret_cast<uint4 *>(ops);
    for (int i = tid; i < sl.nops * 2; i += NT) dst[i] = src[i];
    for (int i = tid; i < sl.ncoef; i += NT) coef[i] = gcoef[sl.coef_off + i];
    for (int i = tid; i < sl.nphase; i += NT) ph[i] = gph[sl.phase_off + i];
    for (int i = tid; i < sl.nent; i += NT) ents[i] = gents[sl.ent_off + i];
    for (int i = tid; i < sl.nterm; i += NT) terms[i] = gterms[sl.term_off + i];
    // deposit tables of the tile base: base(tile) = OR_c btab[c][byte c of tile]
    for (int i = tid; i < 4 * 256; i += NT) {
      const int c = i >> 8;
      uint64_t m = sl.nonactive;
      for (int k = 0; k < 8 * c && m; k++) m &= m - 1;  // drop the lower 8c bits
      btab[i] = pdep64((uint64_t)(i & 255), m);
    }
  }
  __syncthreads();
  for (int p = 0; p < sl.nphase; p++) {
    int rmask = 0;
#pragma unroll
    for (int i = 0; i < RB; i++) rmask |= 1 << ph[p].rbit[i];
    int jt = 0, t = tid, used = rmask;
    if (ph[p].qlane != 0xffff)
      for (int i = 0; i < 4; i++) {
        const int nb = (ph[p].qlane >> (4 * i)) & 15;
        if (nb == 15) break;
        jt |= (t & 1) << nb;
        t >>= 1;
        used |= 1 << nb;
      }
    for (int b = 0; b < K; b++) {
      if ((used >> b) & 1) continue;
      jt |= (t & 1) << b;
      t >>= 1;
    }
    jtab[p * NT + tid] = ((uint32_t)swz<R>(jt) << 16) | (uint32_t)jt;
    uint32_t sa = 0;
    if (ph[p].permuted)
      for (int b = 0; b < K; b++)
        if ((jt >> b) & 1) sa ^= ph[p].colimg[b];
    stab[p * NT + tid] = (uint16_t)sa;
  }
  if (tid < NE) {
    uint64_t o = 0;
#pragma unroll
    for (int i = 0; i < RB; i++)
      if ((tid >> i) & 1) o |= 1ull << sl.act[K - RB + i];
    itoff[tid] = o;
  }
  uint64_t off_t = 0;  // pdep(tid, lowest K-RB active slots)
#pragma unroll
  for (int i = 0; i < K - RB; i++)
    if ((tid >> i) & 1) off_t |= 1ull << sl.act[i];
  const int sw_tid = swz<R>(tid);
  const unsigned sm_base = (unsigned)__cvta_generic_to_shared(buf);
  __syncthreads();

  auto tile_base = [&](uint64_t tile) {
    return btab[tile & 255] | btab[256 + ((tile >> 8) & 255)] | btab[512 + ((tile >> 16) & 255)] |
           btab[768 + ((tile >> 24) & 255)];
  };
  auto issue_load = [&](int bsel, uint64_t base) {
    const T *g = st + base + off_t;
#pragma unroll
    for (int it = 0; it < NE; it++) {
      const unsigned sa = sm_base + (unsigned)((bsel * TILE + (sw_tid ^ swz<R>(it * NT))) * sizeof(T));
      const T *ga = g + itoff[it];
      if (sizeof(T) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(ga));
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(ga));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  const int last = sl.nphase - 1;
  const bool ld = sl.last_direct != 0;
  uint64_t gthr = 0;  // last phase, direct store: this thread's offset
  __shared__ uint64_t limg[4];  // ... and the offsets of its register bits
  if (ld) {
    const int jtl = (int)(jtab[last * NT + tid] & 0xffffu);
    for (int bb = 0; bb < K; bb++)
      if ((jtl >> bb) & 1) gthr ^= sl.lcol[bb];
    if (tid < RB) limg[tid] = sl.lcol[ph[last].rbit[tid]];
    __syncthreads();
  }
  // ring of NBUF tile buffers: the loads of the next NBUF-1 tiles are in
  // flight while a tile is processed (one cp.async group per tile; empty
  // groups keep the group count uniform at the end of the range)
  uint64_t tile = blockIdx.x;
  if (tile >= sl.ntiles) return;
  const uint64_t G = gridDim.x;
#pragma unroll
  for (int k = 0; k < NBUF - 1; k++) {
    const uint64_t t = tile + (uint64_t)k * G;
    if (t < sl.ntiles) issue_load(k, tile_base(t));
    else asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  int b = 0;
  for (; tile < sl.ntiles; tile += G) {
    const uint64_t base = tile_base(tile);
    {
      const uint64_t far = tile + (uint64_t)(NBUF - 1) * G;
      const int fb = (b + NBUF - 1) % NBUF;  // freed at the end of the previous tile
      if (far < sl.ntiles) issue_load(fb, tile_base(far));
      else asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NBUF - 1) : "memory");
    }
    __syncthreads();
    T *tb = buf + b * TILE;
    for (int p = 0; p < sl.nphase; p++) {
      const ShmPhase &P = ph[p];
      const uint32_t jj = jtab[p * NT + tid];
      const int jt = (int)(jj & 0xffffu), sj = (int)(jj >> 16);
      int sr[RB];
#pragma unroll
      for (int i = 0; i < RB; i++) sr[i] = swz<R>(1 << P.rbit[i]);
      T v[NE];
#pragma unroll
      for (int e = 0; e < NE; e++) {
        int a = sj;
#pragma unroll
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) a ^= sr[i];
        v[e] = tb[a];
      }
      for (int oi = P.op_begin; oi < P.op_end; oi++) {
        const ShmOp &o = ops[oi];
        // one 16-byte shared load for the op header (type, t0, t1, flags, ...)
        const uint4 hdr = *reinterpret_cast<const uint4 *>(&o);
        const unsigned otype = hdr.x & 0xffu, oflags = (hdr.x >> 24) & 0xffu;
        if (otype == OP_DIAG) {
          apply_diag<R, RB>(v, o, coef, ents, jt, base);
        } else if (oflags & OPF_FULL) {
          apply_op<R, RB, false>(v, o, coef, true);
        } else {
          if ((base & o.base_mask) != o.base_val) continue;  // tile-uniform
          const bool ok = (jt & o.thr_mask) == o.thr_val;
          if (!__any_sync(0xffffffffu, ok)) continue;
          apply_op<R, RB, true>(v, o, coef, ok);
        }
      }
      if (ld && p == last) {
        // straight to HBM; a permuted map's images overlap, so offsets
        // combine by XOR
        uint64_t cg = gthr;
        if (P.permuted) {
          cg ^= sl.lc0;
          for (int i = P.term_begin; i < P.term_end; i++)
            if ((base & terms[i].base_mask) == terms[i].base_val) cg ^= terms[i].gvec;
        }
#pragma unroll
        for (int e = 0; e < NE; e++) {
          uint64_t o = cg;
#pragma unroll
          for (int i = 0; i < RB; i++)
            if ((e >> i) & 1) o ^= limg[i];
          st[base | o] = v[e];
        }
        break;
      }
      int s0 = sj;
      if (P.permuted) {
        // folded affine permutation: value of tile index j -> A j ^ c(base)
        uint32_t cb = P.c0_swz;
        for (int i = P.term_begin; i < P.term_end; i++)
          if ((base & terms[i].base_mask) == terms[i].base_val) cb ^= terms[i].vec_swz;
        s0 = (int)(stab[p * NT + tid] ^ cb);
#pragma unroll
        for (int i = 0; i < RB; i++) sr[i] = (int)P.colimg[P.rbit[i]];
        __syncthreads();  // every thread has read its elements before any permuted store
      }
#pragma unroll
      for (int e = 0; e < NE; e++) {
        int a = s0;
#pragma unroll
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) a ^= sr[i];
        tb[a] = v[e];
      }
      __syncthreads();
    }
    if (!ld) {
      const T *tbc = tb;
      T *g = st + base + off_t;
#pragma unroll
      for (int it = 0; it < NE; it++) g[itoff[it]] = tbc[sw_tid ^ swz<R>(it * NT)];
    }
    __syncthreads();  // the buffer is free for the next load
    b = (b + 1) % NBUF;
  }
}

// ---------------------------------------------------------- permute / misc
template <typename T>
__global__ void __launch_bounds__(256) permute_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                      uint64_t N, uint64_t src_mask, int nmoved,
                                                      int4 mv0, int4 mv1, int4 mv2) {
  // mvK = {src0, dst0, src1, dst1}: up to 6 moved bits
  const int src[6] = {mv0.x, mv0.z, mv1.x, mv1.z, mv2.x, mv2.z};
  const int dst[6] = {mv0.y, mv0.w, mv1.y, mv1.w, mv2.y, mv2.w};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    uint64_t o = i & ~src_mask;
#pragma unroll
    for (int b = 0; b < 6; b++)
      if (b < nmoved) o |= ((i >> src[b]) & 1ull) << dst[b];
    out[o] = in[i];
  }
}

// general permutation: out[newpos(i)] = in[i] with an arbitrary slot map
template <typename T>
__global__ void __launch_bounds__(256) permute_general_kernel(const T *__restrict__ in,
                                                              T *__restrict__ out, uint64_t N,
                                                              const int *__restrict__ newpos,
                                                              int L) {
  __shared__ int np[64];
  if (threadIdx.x < 64) np[threadIdx.x] = threadIdx.x < L ? newpos[threadIdx.x] : 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    uint64_t o = 0;
    for (int b = 0; b < L; b++) o |= ((i >> b) & 1ull) << np[b];
    out[o] = in[i];
  }
}

// ---------------------------------------------- in-place remap (NEXT-3)
// At HBM capacity there is no second shard buffer (n = 36 fp64 on 8 GPUs:
// 128 GiB per shard), so the remap of P:L1312 / P:L1367-1371 runs in place
// as a sequence of pair swaps, each a single pass with no scratch:
//  * swap_bits_kernel: transposition of index bits a < b, i.e. the pairs
//    (x with a=1,b=0) <-> (x with a=0,b=1) -- any local bit permutation
//    (the "pack") is a product of at most L-1 of them;
//  * xor_swap_kernel: x <-> x ^ F for every x whose lowest set bit of F is 0
//    (the block relabelling that resolves the flips of incoming qubits);
//  * swap_regions_kernel: a[i] <-> b[i] (the block exchange between two
//    shards of a virtual world on one GPU).
// 128-bit loads and stores; a grid-stride loop over the pairs.
template <typename T>
__global__ void __launch_bounds__(256) swap_bits_kernel(T *__restrict__ st, uint64_t npairs, int a, int b) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lo_a = (1ull << a) - 1, lo_b = (1ull << b) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
    // deposit i around bit positions a < b (both 0), then set a
    uint64_t x = (i & lo_a) | ((i & ~lo_a) << 1);
    x = (x & lo_b) | ((x & ~lo_b) << 1);
    x |= 1ull << a;
    const uint64_t y = x ^ (1ull << a) ^ (1ull << b);
    const T u = st[x], v = st[y];
    st[x] = v;
    st[y] = u;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) xor_swap_kernel(T *__restrict__ st, uint64_t npairs, uint64_t F,
                                                       int low) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lo = (1ull << low) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
    const uint64_t x = (i & lo) | ((i & ~lo) << 1);  // bit `low` = 0
    const uint64_t y = x ^ F;
    const T u = st[x], v = st[y];
    st[x] = v;
    st[y] = u;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) swap_regions_kernel(T *__restrict__ a, T *__restrict__ b, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T u = a[i], v = b[i];
    a[i] = v;
    b[i] = u;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) scale_kernel(T *__restrict__ st, uint64_t N, double re,
                                                    double im) {
  T s;
  s.x = re;
  s.y = im;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride)
    st[i] = cmul(s, st[i]);
}

template <typename T>
__global__ void init_one_kernel(T *st) {
  T one;
  one.x = 1;
  one.y = 0;
  st[0] = one;
}

// ----------------------------------------------------------- host launchers
static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <typename R, int k>
static cudaError_t launch_fused_k(void *st, int L, const FusedLaunch &fl, const double2 *mats,
                                  cudaStream_t s) {
  using T = typename Cplx<R>::T;
  const uint64_t ngroups = 1ull << (L - k);
  const int threads = 256;
  const size_t smem = sizeof(T) << (2 * k);
  auto kern = fused_kernel<R, k>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  uint64_t want = (ngroups + threads - 1) / threads;
  uint64_t cap = (uint64_t)num_sms() * 16;
  int grid = (int)(want < cap ? want : cap);
  if (grid < 1) grid = 1;
  kern<<<grid, threads, smem, s>>>((T *)st, ngroups, fl, mats);
  return cudaGetLastError();
}

template <typename R>
static cudaError_t launch_fused_t(void *st, int L, const FusedLaunch &fl, const double2 *mats,
                                  cudaStream_t s) {
  switch (fl.k) {
    case 1: return launch_fused_k<R, 1>(st, L, fl, mats, s);
    case 2: return launch_fused_k<R, 2>(st, L, fl, mats, s);
    case 3: return launch_fused_k<R, 3>(st, L, fl, mats, s);
    case 4: return launch_fused_k<R, 4>(st, L, fl, mats, s);
    case 5: return launch_fused_k<R, 5>(st, L, fl, mats, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fused(int dtype, void *st, int L, const FusedLaunch &fl, const double2 *mats,
                         cudaStream_t s) {
  return dtype == 0 ? launch_fused_t<double>(st, L, fl, mats, s)
                    : launch_fused_t<float>(st, L, fl, mats, s);
}

template <typename R, int K, int RB, int NBUF>
static cudaError_t launch_shm_k(void *st, const ShmLaunch &sl, const ShmOp *ops,
                                const double *coef, const ShmPhase *ph, const DiagEnt *ents,
                                const PermTerm *terms, cudaStream_t s) {
  using T = typename Cplx<R>::T;
  constexpr int NT = 1 << (K - RB);
  const ShmSmem lay = shm_smem_layout((int)sizeof(T) << K, NBUF, sl, NT, 1 << RB);
  auto kern = shm_kernel<R, K, RB, NBUF>;
  static int attr_set = 0;
  if (attr_set < (int)lay.total) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lay.total);
    if (e != cudaSuccess) return e;
    attr_set = (int)lay.total;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, lay.total);
  if (occ < 1) occ = 1;
  uint64_t grid = (uint64_t)num_sms() * occ;
  if (grid > sl.ntiles) grid = sl.ntiles;
  if (sl.grid_cap > 0 && grid > (uint64_t)sl.grid_cap) grid = (uint64_t)sl.grid_cap;
  kern<<<(unsigned)grid, NT, lay.total, s>>>((T *)st, sl, ops, coef, ph, ents, terms);
  return cudaGetLastError();
}

// tile configuration: (K, RB, NBUF).  Double buffering while two tiles fit.
template <typename R>
static cudaError_t launch_shm_t(void *st, const ShmLaunch &sl, const ShmOp *ops,
                                const double *coef, const ShmPhase *ph, const DiagEnt *ents,
                                const PermTerm *terms, cudaStream_t s) {
  constexpr bool F64 = sizeof(R) == 8;
  switch (sl.K) {
    case 6: return launch_shm_k<R, 6, 1, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 7: return launch_shm_k<R, 7, 2, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 8: return launch_shm_k<R, 8, 3, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 9: return launch_shm_k<R, 9, 4, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 10: return launch_shm_k<R, 10, 4, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 11: return sl.nbuf == 1 ? launch_shm_k<R, 11, 4, 1>(st, sl, ops, coef, ph, ents, terms, s)
                                : launch_shm_k<R, 11, 4, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 12:
      if (sl.RB == 3) return launch_shm_k<R, 12, 3, 1>(st, sl, ops, coef, ph, ents, terms, s);
      // three tile buffers only while they fit the 227 KiB opt-in limit
      if (sl.nbuf == 3 &&
          shm_smem_layout((int)sizeof(typename Cplx<R>::T) << 12, 3, sl, 256, 16).total <= 232448)
        return launch_shm_k<R, 12, 4, 3>(st, sl, ops, coef, ph, ents, terms, s);
      return sl.nbuf == 1 ? launch_shm_k<R, 12, 4, 1>(st, sl, ops, coef, ph, ents, terms, s)
                          : launch_shm_k<R, 12, 4, 2>(st, sl, ops, coef, ph, ents, terms, s);
    case 13: return (F64 || sl.nbuf == 1) ? launch_shm_k<R, 13, 4, 1>(st, sl, ops, coef, ph, ents, terms, s)
                        : launch_shm_k<R, 13, 4, 2>(st, sl, ops, coef, ph, ents, terms, s);
  }
  return cudaErrorInvalidValue;
}

int shm_register_bits(int K) { return K >= 9 ? 4 : K - 5; }

// number of tile buffers launch_shm_t picks for a launch (jit.cpp mirrors it)
int shm_nbuf_effective(int dtype, const ShmLaunch &sl) {
  const bool F64 = dtype == 0;
  if (sl.K <= 10) return 2;
  if (sl.K == 11) return sl.nbuf == 1 ? 1 : 2;
  if (sl.K == 12) {
    if (sl.RB == 3) return 1;
    const int esz = F64 ? 16 : 8;
    if (sl.nbuf == 3 && shm_smem_layout(esz << 12, 3, sl, 256, 16).total <= 232448) return 3;
    return sl.nbuf == 1 ? 1 : 2;
  }
  return (F64 || sl.nbuf == 1) ? 1 : 2;
}

cudaError_t launch_shm(int dtype, void *st, const ShmLaunch &sl, const ShmOp *ops,
                       const double *coef, const ShmPhase *ph, const DiagEnt *ents,
                       const PermTerm *terms, cudaStream_t s) {
  return dtype == 0 ? launch_shm_t<double>(st, sl, ops, coef, ph, ents, terms, s)
                    : launch_shm_t<float>(st, sl, ops, coef, ph, ents, terms, s);
}

cudaError_t launch_permute(int dtype, const void *in, void *out, int L, const int *newpos_host,
                           const int *newpos_dev, cudaStream_t s) {
  const uint64_t N = 1ull << L;
  int src[6], dst[6], nm = 0;
  uint64_t smask = 0;
  bool general = false;
  for (int b = 0; b < L; b++) {
    if (newpos_host[b] == b) continue;
    if (nm == 6) { general = true; break; }
    src[nm] = b;
    dst[nm] = newpos_host[b];
    smask |= 1ull << b;
    nm++;
  }
  for (int i = nm; i < 6; i++) src[i] = dst[i] = 0;
  const int threads = 256;
  uint64_t want = (N + threads - 1) / threads;
  uint64_t cap = (uint64_t)num_sms() * 32;
  int grid = (int)(want < cap ? want : cap);
  if (general) {
    if (dtype == 0)
      permute_general_kernel<double2><<<grid, threads, 0, s>>>((const double2 *)in, (double2 *)out, N, newpos_dev, L);
    else
      permute_general_kernel<float2><<<grid, threads, 0, s>>>((const float2 *)in, (float2 *)out, N, newpos_dev, L);
  } else {
    int4 a = {src[0], dst[0], src[1], dst[1]}, b = {src[2], dst[2], src[3], dst[3]},
         c = {src[4], dst[4], src[5], dst[5]};
    if (dtype == 0)
      permute_kernel<double2><<<grid, threads, 0, s>>>((const double2 *)in, (double2 *)out, N, smask, nm, a, b, c);
    else
      permute_kernel<float2><<<grid, threads, 0, s>>>((const float2 *)in, (float2 *)out, N, smask, nm, a, b, c);
  }
  return cudaGetLastError();
}

static int pair_grid(uint64_t n) {
  const uint64_t want = (n + 255) / 256, cap = (uint64_t)num_sms() * 32;
  return (int)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_swap_bits(int dtype, void *st, int L, int a, int b, cudaStream_t s) {
  if (a == b) return cudaSuccess;
  if (a > b) std::swap(a, b);
  const uint64_t np = 1ull << (L - 2);
  if (dtype == 0) swap_bits_kernel<double2><<<pair_grid(np), 256, 0, s>>>((double2 *)st, np, a, b);
  else swap_bits_kernel<float2><<<pair_grid(np), 256, 0, s>>>((float2 *)st, np, a, b);
  return cudaGetLastError();
}

cudaError_t launch_xor_swap(int dtype, void *st, int L, uint64_t F, cudaStream_t s) {
  if (!F) return cudaSuccess;
  const uint64_t np = 1ull << (L - 1);
  const int low = __builtin_ctzll(F);
  if (dtype == 0) xor_swap_kernel<double2><<<pair_grid(np), 256, 0, s>>>((double2 *)st, np, F, low);
  else xor_swap_kernel<float2><<<pair_grid(np), 256, 0, s>>>((float2 *)st, np, F, low);
  return cudaGetLastError();
}

cudaError_t launch_swap_regions(int dtype, void *a, void *b, uint64_t n, cudaStream_t s) {
  if (!n) return cudaSuccess;
  if (dtype == 0) swap_regions_kernel<double2><<<pair_grid(n), 256, 0, s>>>((double2 *)a, (double2 *)b, n);
  else swap_regions_kernel<float2><<<pair_grid(n), 256, 0, s>>>((float2 *)a, (float2 *)b, n);
  return cudaGetLastError();
}

cudaError_t launch_scale(int dtype, void *st, int L, double re, double im, cudaStream_t s) {
  const uint64_t N = 1ull << L;
  const int threads = 256;
  uint64_t want = (N + threads - 1) / threads;
  uint64_t cap = (uint64_t)num_sms() * 32;
  int grid = (int)(want < cap ? want : cap);
  if (dtype == 0)
    scale_kernel<double2><<<grid, threads, 0, s>>>((double2 *)st, N, re, im);
  else
    scale_kernel<float2><<<grid, threads, 0, s>>>((float2 *)st, N, re, im);
  return cudaGetLastError();
}

cudaError_t launch_init(int dtype, void *st, int L, bool one, cudaStream_t s) {
  const size_t bytes = (dtype == 0 ? (size_t)16 : (size_t)8) << L;
  cudaError_t e = cudaMemsetAsync(st, 0, bytes, s);
  if (e != cudaSuccess || !one) return e;
  if (dtype == 0)
    init_one_kernel<double2><<<1, 1, 0, s>>>((double2 *)st);
  else
    init_one_kernel<float2><<<1, 1, 0, s>>>((float2 *)st);
  return cudaGetLastError();
}

}  // namespace atlas
