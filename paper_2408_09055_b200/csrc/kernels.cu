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
#include <cuda_runtime.h>

#include <cstdint>

#include "device.h"

namespace atlas {

template <typename R> struct Cplx;
template <> struct Cplx<double> { using T = double2; };
template <> struct Cplx<float> { using T = float2; };

// ------------------------------------------------------------------ helpers
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

// Swizzle of a tile index so that the 8 (fp64) / 16 (fp32) lanes of one
// shared-memory wavefront hit distinct 16-byte bank groups for the access
// patterns of the load/store loops and of most register phases.
template <typename R> __device__ __forceinline__ int swz(int j);
template <> __device__ __forceinline__ int swz<double>(int j) {
  return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9) ^ (j >> 12)) & 7);
}
template <> __device__ __forceinline__ int swz<float>(int j) {
  return j ^ (((j >> 4) ^ (j >> 8) ^ (j >> 12)) & 15);
}

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
template <typename T, int NE, int TB>
__device__ __forceinline__ void dense1(T (&v)[NE], const T (&m)[4], int need_mask,
                                       int need_val, bool fixed_ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & (1 << TB)) continue;
    const int e1 = e | (1 << TB);
    if (fixed_ok && (e & need_mask) == need_val) {
      T a = v[e], b = v[e1];
      T y0, y1;
      y0.x = 0; y0.y = 0; y1.x = 0; y1.y = 0;
      cmac(y0, m[0], a);
      cmac(y0, m[1], b);
      cmac(y1, m[2], a);
      cmac(y1, m[3], b);
      v[e] = y0;
      v[e1] = y1;
    }
  }
}

template <typename T, int NE, int TB>
__device__ __forceinline__ void perm1(T (&v)[NE], int need_mask, int need_val, bool fixed_ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & (1 << TB)) continue;
    const int e1 = e | (1 << TB);
    if (fixed_ok && (e & need_mask) == need_val) {
      T a = v[e];
      v[e] = v[e1];
      v[e1] = a;
    }
  }
}

template <typename T, int NE, int TB0, int TB1>
__device__ __forceinline__ void dense2(T (&v)[NE], const double *__restrict__ m, int need_mask,
                                       int need_val, bool fixed_ok) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (e & ((1 << TB0) | (1 << TB1))) continue;
    if (fixed_ok && (e & need_mask) == need_val) {
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

template <typename R, int RB>
__device__ __forceinline__ void apply_op(typename Cplx<R>::T (&v)[1 << RB],
                                         const ShmOp *__restrict__ op, int jt, uint64_t base) {
  using T = typename Cplx<R>::T;
  constexpr int NE = 1 << RB;
  const int type = op->type;
  const int nsel = op->nsel;
  // Split the selector into its register part (varies per element) and its
  // fixed part (thread bits of the tile, or non-active bits of the tile base).
  int reg_mask = 0, reg_bit_of_sel[3] = {0, 0, 0};
  int fixed = 0, fixed_mask = 0;
  for (int s = 0; s < nsel; s++) {
    const int src = op->sel_src[s], idx = op->sel_idx[s];
    if (src == SEL_REG) {
      reg_mask |= 1 << idx;
      reg_bit_of_sel[s] = idx;
    } else {
      const int bitv = (src == SEL_THR) ? ((jt >> idx) & 1) : (int)((base >> idx) & 1);
      fixed |= bitv << s;
      fixed_mask |= 1 << s;
    }
  }
  if (type == OP_DIAG) {
    // y = ph[sel] * x; loop over selector values (<= 8)
    const int nv = 1 << nsel;
    for (int sv = 0; sv < nv; sv++) {
      if ((sv & fixed_mask) != fixed) continue;
      T ph;
      ph.x = (R)op->m[2 * sv];
      ph.y = (R)op->m[2 * sv + 1];
      if (ph.x == (R)1 && ph.y == (R)0) continue;
      int need = 0;
      for (int s = 0; s < nsel; s++)
        if ((reg_mask >> reg_bit_of_sel[s]) & 1 && op->sel_src[s] == SEL_REG)
          need |= ((sv >> s) & 1) << reg_bit_of_sel[s];
#pragma unroll
      for (int e = 0; e < NE; e++)
        if ((e & reg_mask) == need) v[e] = cmul(ph, v[e]);
    }
    return;
  }
  const int selv = op->selv;
  const bool fixed_ok = (selv & fixed_mask) == fixed;
  if (!__any_sync(0xffffffffu, fixed_ok)) return;
  int need = 0;
  for (int s = 0; s < nsel; s++)
    if (op->sel_src[s] == SEL_REG) need |= ((selv >> s) & 1) << reg_bit_of_sel[s];
  const int t0 = op->t0;
  if (type == OP_PERM1) {
    switch (t0) {
      case 0: perm1<T, NE, 0>(v, reg_mask, need, fixed_ok); break;
      case 1: if (RB > 1) perm1<T, NE, (RB > 1 ? 1 : 0)>(v, reg_mask, need, fixed_ok); break;
      case 2: if (RB > 2) perm1<T, NE, (RB > 2 ? 2 : 0)>(v, reg_mask, need, fixed_ok); break;
      case 3: if (RB > 3) perm1<T, NE, (RB > 3 ? 3 : 0)>(v, reg_mask, need, fixed_ok); break;
    }
    return;
  }
  if (type == OP_DENSE1) {
    T m[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      m[i].x = (R)op->m[2 * i];
      m[i].y = (R)op->m[2 * i + 1];
    }
    switch (t0) {
      case 0: dense1<T, NE, 0>(v, m, reg_mask, need, fixed_ok); break;
      case 1: if (RB > 1) dense1<T, NE, (RB > 1 ? 1 : 0)>(v, m, reg_mask, need, fixed_ok); break;
      case 2: if (RB > 2) dense1<T, NE, (RB > 2 ? 2 : 0)>(v, m, reg_mask, need, fixed_ok); break;
      case 3: if (RB > 3) dense1<T, NE, (RB > 3 ? 3 : 0)>(v, m, reg_mask, need, fixed_ok); break;
    }
    return;
  }
  // OP_DENSE2, t0 < t1
  const int code = op->t0 * 4 + op->t1;
  const double *m = op->m;
  switch (code) {
    case 1: if (RB > 1) dense2<T, NE, 0, (RB > 1 ? 1 : 0)>(v, m, reg_mask, need, fixed_ok); break;
    case 2: if (RB > 2) dense2<T, NE, 0, (RB > 2 ? 2 : 0)>(v, m, reg_mask, need, fixed_ok); break;
    case 3: if (RB > 3) dense2<T, NE, 0, (RB > 3 ? 3 : 0)>(v, m, reg_mask, need, fixed_ok); break;
    case 6: if (RB > 2) dense2<T, NE, (RB > 2 ? 1 : 0), (RB > 2 ? 2 : 0)>(v, m, reg_mask, need, fixed_ok); break;
    case 7: if (RB > 3) dense2<T, NE, (RB > 3 ? 1 : 0), (RB > 3 ? 3 : 0)>(v, m, reg_mask, need, fixed_ok); break;
    case 11: if (RB > 3) dense2<T, NE, (RB > 3 ? 2 : 0), (RB > 3 ? 3 : 0)>(v, m, reg_mask, need, fixed_ok); break;
  }
}

template <typename R, int K, int RB>
__global__ void __launch_bounds__(1 << (K - RB)) shm_kernel(
    typename Cplx<R>::T *__restrict__ st, ShmLaunch sl, const uint64_t *__restrict__ hightab,
    const ShmOp *__restrict__ ops, const ShmPhase *__restrict__ phases) {
  using T = typename Cplx<R>::T;
  constexpr int NT = 1 << (K - RB);
  constexpr int NE = 1 << RB;
  constexpr int TILE = 1 << K;
  extern __shared__ unsigned char smraw[];
  T *sm = reinterpret_cast<T *>(smraw);
  const int tid = threadIdx.x;
  const int c0 = sl.c0;
  const int lowmask = (1 << c0) - 1;
  const uint64_t *ht = hightab + sl.hightab_off;
  const ShmOp *op0 = ops + sl.ops_off;
  const ShmPhase *ph0 = phases + sl.phase_off;

  for (uint64_t tile = blockIdx.x; tile < sl.ntiles; tile += gridDim.x) {
    const uint64_t base = pdep64(tile, sl.nonactive);
    // HBM -> SMEM: element j = it * NT + tid; consecutive threads read
    // consecutive amplitudes inside runs of 2^c0 (c0 >= 5: 512 B for fp64).
#pragma unroll
    for (int it = 0; it < NE; it++) {
      const int j = it * NT + tid;
      const uint64_t off = (uint64_t)(j & lowmask) | ht[j >> c0];
      cp_async(&sm[swz<R>(j)], &st[base + off]);
    }
    cp_async_wait_all();
    __syncthreads();
    for (int p = 0; p < sl.nphase; p++) {
      const ShmPhase P = ph0[p];
      int rmask = 0;
#pragma unroll
      for (int i = 0; i < RB; i++) rmask |= 1 << P.rbit[i];
      // thread part of the tile index: deposit tid into the non-register bits
      int jt = 0;
      {
        int t = tid;
        for (int b = 0; b < K; b++) {
          if ((rmask >> b) & 1) continue;
          jt |= (t & 1) << b;
          t >>= 1;
        }
      }
      int rv[RB];
#pragma unroll
      for (int i = 0; i < RB; i++) rv[i] = 1 << P.rbit[i];
      T v[NE];
#pragma unroll
      for (int e = 0; e < NE; e++) {
        int j = jt;
#pragma unroll
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) j |= rv[i];
        v[e] = sm[swz<R>(j)];
      }
      for (int o = P.op_begin; o < P.op_end; o++) apply_op<R, RB>(v, op0 + o, jt, base);
#pragma unroll
      for (int e = 0; e < NE; e++) {
        int j = jt;
#pragma unroll
        for (int i = 0; i < RB; i++)
          if ((e >> i) & 1) j |= rv[i];
        sm[swz<R>(j)] = v[e];
      }
      __syncthreads();
    }
    // SMEM -> HBM, same coalesced pattern as the load
#pragma unroll
    for (int it = 0; it < NE; it++) {
      const int j = it * NT + tid;
      const uint64_t off = (uint64_t)(j & lowmask) | ht[j >> c0];
      st[base + off] = sm[swz<R>(j)];
    }
    __syncthreads();
  }
  (void)TILE;
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

template <typename R, int K, int RB>
static cudaError_t launch_shm_k(void *st, const ShmLaunch &sl, const uint64_t *ht,
                                const ShmOp *ops, const ShmPhase *ph, cudaStream_t s) {
  using T = typename Cplx<R>::T;
  const size_t smem = sizeof(T) << K;
  auto kern = shm_kernel<R, K, RB>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  uint64_t grid = sl.ntiles;
  const uint64_t cap = (uint64_t)1 << 30;
  if (grid > cap) grid = cap;
  kern<<<(unsigned)grid, 1 << (K - RB), smem, s>>>((T *)st, sl, ht, ops, ph);
  return cudaGetLastError();
}

template <typename R>
static cudaError_t launch_shm_t(void *st, const ShmLaunch &sl, const uint64_t *ht,
                                const ShmOp *ops, const ShmPhase *ph, cudaStream_t s) {
  switch (sl.K) {
    case 6: return launch_shm_k<R, 6, 1>(st, sl, ht, ops, ph, s);
    case 7: return launch_shm_k<R, 7, 2>(st, sl, ht, ops, ph, s);
    case 8: return launch_shm_k<R, 8, 3>(st, sl, ht, ops, ph, s);
    case 9: return launch_shm_k<R, 9, 4>(st, sl, ht, ops, ph, s);
    case 10: return launch_shm_k<R, 10, 4>(st, sl, ht, ops, ph, s);
    case 11: return launch_shm_k<R, 11, 4>(st, sl, ht, ops, ph, s);
    case 12: return launch_shm_k<R, 12, 4>(st, sl, ht, ops, ph, s);
    case 13: return launch_shm_k<R, 13, 4>(st, sl, ht, ops, ph, s);
  }
  return cudaErrorInvalidValue;
}

int shm_register_bits(int K) { return K >= 9 ? 4 : K - 5; }

cudaError_t launch_shm(int dtype, void *st, const ShmLaunch &sl, const uint64_t *ht,
                       const ShmOp *ops, const ShmPhase *ph, cudaStream_t s) {
  return dtype == 0 ? launch_shm_t<double>(st, sl, ht, ops, ph, s)
                    : launch_shm_t<float>(st, sl, ht, ops, ph, s);
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
  const size_t bytes = (dtype == 0 ? 16 : 8) << L;
  cudaError_t e = cudaMemsetAsync(st, 0, bytes, s);
  if (e != cudaSuccess || !one) return e;
  if (dtype == 0)
    init_one_kernel<double2><<<1, 1, 0, s>>>((double2 *)st);
  else
    init_one_kernel<float2><<<1, 1, 0, s>>>((float2 *)st);
  return cudaGetLastError();
}

}  // namespace atlas
