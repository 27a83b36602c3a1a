// runtime.cu -- Execute (Alg. 1) and the C-ABI.
//
// Per stage: Shard (the inter-stage remap: optional local bit-permutation
// "pack", then the all-to-all exchange of contiguous blocks -- NCCL grouped
// send/recv over NVLink, or device copies in virtual-world mode) followed by
// LaunchKernel for every kernel of the stage on this rank's 2^L shard
// ("ParFor shard": every rank runs its own shard; no collective
// inside a stage).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>

#include "ctx.h"

namespace atlas {

void build_plan(atlas_ctx *C, int s_max, double cf);
std::string plan_json(const atlas_ctx *C);
cudaError_t launch_fused(int dtype, void *st, int L, const FusedLaunch &fl, const double2 *mats,
                         cudaStream_t s);
cudaError_t launch_shm(int dtype, void *st, const ShmLaunch &sl, const ShmOp *ops,
                       const double *coef, const ShmPhase *ph, const DiagEnt *ents,
                       const PermTerm *terms, cudaStream_t s);
cudaError_t launch_permute(int dtype, const void *in, void *out, int L, const int *newpos_host,
                           const int *newpos_dev, cudaStream_t s);
cudaError_t launch_scale(int dtype, void *st, int L, double re, double im, cudaStream_t s);
cudaError_t launch_swap_bits(int dtype, void *st, int L, int a, int b, cudaStream_t s);
cudaError_t launch_xor_swap(int dtype, void *st, int L, uint64_t F, cudaStream_t s);
cudaError_t launch_swap_regions(int dtype, void *a, void *b, uint64_t n, cudaStream_t s);
cudaError_t launch_init(int dtype, void *st, int L, bool one, cudaStream_t s);
void shm_jit_prepare(atlas_ctx *C);
cudaError_t launch_shm_jit(void *jit, void *st, void *dst, const ShmLaunch &sl, cudaStream_t s, int zmode,
                           uint64_t skip, void *const *peers, uint64_t zq);
bool shm_jit_zero_ok(const void *jit);

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) fail(ATLAS_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_));       \
  } while (0)

// ------------------------------------------------------------------- NCCL
// libnccl.so.2 is loaded at run time (torch ships NCCL 2.28); only the few
// entry points the remap needs are bound.
struct NcclApi {
  void *h = nullptr;
  int (*getUniqueId)(void *) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*commDestroy)(void *) = nullptr;
  int (*allGather)(const void *, void *, size_t, int, void *, cudaStream_t) = nullptr;
  int (*allReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  const char *(*errStr)(int) = nullptr;
  void *commInitRank = nullptr;
};
struct Uid {
  char internal[128];
};
static NcclApi g_nccl;
static std::mutex g_nccl_mu;

void nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *nm : names) {
    g_nccl.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) fail(ATLAS_E_NCCL, "cannot load libnccl.so.2: %s", dlerror());
  g_nccl.getUniqueId = (int (*)(void *))dlsym(g_nccl.h, "ncclGetUniqueId");
  g_nccl.groupStart = (int (*)())dlsym(g_nccl.h, "ncclGroupStart");
  g_nccl.groupEnd = (int (*)())dlsym(g_nccl.h, "ncclGroupEnd");
  g_nccl.send = (int (*)(const void *, size_t, int, int, void *, cudaStream_t))dlsym(g_nccl.h, "ncclSend");
  g_nccl.recv = (int (*)(void *, size_t, int, int, void *, cudaStream_t))dlsym(g_nccl.h, "ncclRecv");
  g_nccl.commDestroy = (int (*)(void *))dlsym(g_nccl.h, "ncclCommDestroy");
  g_nccl.allGather = (int (*)(const void *, void *, size_t, int, void *, cudaStream_t))dlsym(g_nccl.h, "ncclAllGather");
  g_nccl.allReduce =
      (int (*)(const void *, void *, size_t, int, int, void *, cudaStream_t))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.errStr = (const char *(*)(int))dlsym(g_nccl.h, "ncclGetErrorString");
  g_nccl.commInitRank = dlsym(g_nccl.h, "ncclCommInitRank");
  if (!g_nccl.getUniqueId || !g_nccl.groupStart || !g_nccl.groupEnd || !g_nccl.send ||
      !g_nccl.recv || !g_nccl.commInitRank)
    fail(ATLAS_E_NCCL, "libnccl.so.2 lacks required symbols");
}

#define NK(x)                                                                         \
  do {                                                                                \
    int r_ = (x);                                                                     \
    if (r_ != 0)                                                                      \
      fail(ATLAS_E_NCCL, "%s: %s", #x, g_nccl.errStr ? g_nccl.errStr(r_) : "error");  \
  } while (0)

static const int kNcclUint8 = 1;  // ncclUint8 (nccl.h)
static const int kNcclInt32 = 2;  // ncclInt32
static const int kNcclSum = 0;    // ncclSum
static const int kNcclMin = 3;    // ncclMin

// ---------------------------------------------------------------- device
static size_t amp_bytes(const atlas_ctx *C) { return C->dt == ATLAS_C128 ? 16 : 8; }
static size_t shard_bytes(const atlas_ctx *C) { return amp_bytes(C) << C->L; }

void ensure_device(atlas_ctx *C) {
  if (C->dev_ready) return;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) fail(ATLAS_E_CUDA, "no CUDA device available");
  if (C->opt.device >= 0) C->device = C->opt.device;
  else CK(cudaGetDevice(&C->device));
  CK(cudaSetDevice(C->device));
  if (!C->stream) {
    CK(cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking));
    C->own_stream = true;
  }
  const int slots = C->nslots;
  C->cur.assign(slots, 0);
  if (C->offload) {
    // two pinned host copies of the whole state (stage ping-pong) and two
    // device work shards (the second receives a fused pack's output)
    const size_t hb = amp_bytes(C) << C->n;
    for (int i = 0; i < 2; i++) {
      if (cudaHostAlloc(&C->h_buf[i], hb, cudaHostAllocDefault) != cudaSuccess)
        fail(ATLAS_E_OOM, "cudaHostAlloc(%zu) offload host buffer failed", hb);
      if (cudaMalloc(&C->d_work[i], shard_bytes(C)) != cudaSuccess)
        fail(ATLAS_E_OOM, "cudaMalloc(%zu) offload work shard failed", shard_bytes(C));
    }
    C->d_state.assign(slots, nullptr);
    C->d_scratch.assign(slots, nullptr);
    C->dev_ready = true;
    return;
  }
  if (!C->bound) {
    C->d_state.assign(slots, nullptr);
    C->d_scratch.assign(slots, nullptr);
    const size_t b = shard_bytes(C);
    for (int s = 0; s < slots; s++) {
      if (cudaMalloc(&C->d_state[s], b) != cudaSuccess)
        fail(ATLAS_E_OOM, "cudaMalloc(%zu) state failed", b);
      if (C->world > 1 && !C->opt.inplace_remap && cudaMalloc(&C->d_scratch[s], b) != cudaSuccess)
        fail(ATLAS_E_OOM, "cudaMalloc(%zu) scratch failed", b);
    }
  }
  if (C->world > 1 && !C->opt.virtual_world && !C->nccl_comm) {
    nccl_load();
    if (!C->have_uid) fail(ATLAS_E_INVALID, "world > 1 needs an nccl_uid (or virtual_world)");
    Uid u;
    memcpy(u.internal, C->nccl_uid, 128);
    auto init = (int (*)(void **, int, Uid, int))g_nccl.commInitRank;
    NK(init(&C->nccl_comm, C->world, u, C->rank));
  }
  // fused exchange over peer memory: every rank opens every other rank's
  // state and scratch shard (CUDA IPC handles allgathered over NCCL); the
  // last shared-memory launch of a stage then stores each packed block
  // straight into its destination rank's buffer over NVLink, and an
  // allreduce of 4 bytes ends the exchange (library-owned buffers only)
  if (C->world > 1 && C->nslots == 1 && C->nccl_comm && C->opt.shm_fuse_exchange && !C->opt.inplace_remap &&
      !C->bound && !C->ipc_ready && g_nccl.allGather && g_nccl.allReduce) {
    const int W = C->world;
    // every rank must agree on using peer memory (a rank that could not
    // open a peer's buffers makes all of them keep the NCCL exchange)
    int ok = 1;
    cudaIpcMemHandle_t h[2];
    if (cudaIpcGetMemHandle(&h[0], C->d_state[0]) != cudaSuccess ||
        cudaIpcGetMemHandle(&h[1], C->d_scratch[0]) != cudaSuccess) {
      ok = 0;
      memset(h, 0, sizeof h);
    }
    void *d_h = nullptr;
    CK(cudaMalloc(&d_h, (size_t)(W + 1) * sizeof h + 8));
    CK(cudaMemcpy(d_h, h, sizeof h, cudaMemcpyHostToDevice));
    NK(g_nccl.allGather(d_h, (char *)d_h + sizeof h, sizeof h, kNcclUint8, C->nccl_comm, C->stream));
    std::vector<cudaIpcMemHandle_t> all(2 * (size_t)W);
    CK(cudaMemcpyAsync(all.data(), (char *)d_h + sizeof h, (size_t)W * sizeof h, cudaMemcpyDeviceToHost,
                       C->stream));
    CK(cudaStreamSynchronize(C->stream));
    C->ipc_state.assign(W, nullptr);
    C->ipc_scratch.assign(W, nullptr);
    for (int r = 0; r < W && ok; r++) {
      if (r == C->rank) {
        C->ipc_state[r] = C->d_state[0];
        C->ipc_scratch[r] = C->d_scratch[0];
        continue;
      }
      if (cudaIpcOpenMemHandle(&C->ipc_state[r], all[2 * r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
          cudaIpcOpenMemHandle(&C->ipc_scratch[r], all[2 * r + 1], cudaIpcMemLazyEnablePeerAccess) !=
              cudaSuccess)
        ok = 0;
    }
    cudaGetLastError();  // a failed open is handled by the agreement below
    int *d_ok = (int *)((char *)d_h + (size_t)(W + 1) * sizeof h);
    CK(cudaMemcpy(d_ok, &ok, 4, cudaMemcpyHostToDevice));
    NK(g_nccl.allReduce(d_ok, d_ok, 1, kNcclInt32, kNcclMin, C->nccl_comm, C->stream));
    CK(cudaMemcpyAsync(&ok, d_ok, 4, cudaMemcpyDeviceToHost, C->stream));
    CK(cudaStreamSynchronize(C->stream));
    cudaFree(d_h);
    if (ok) {
      CK(cudaMalloc(&C->d_bar, 4));
      CK(cudaMemset(C->d_bar, 0, 4));
      C->ipc_ready = true;
    } else {
      for (int r = 0; r < W; r++)
        if (r != C->rank) {
          if (C->ipc_state[r]) cudaIpcCloseMemHandle(C->ipc_state[r]);
          if (C->ipc_scratch[r]) cudaIpcCloseMemHandle(C->ipc_scratch[r]);
        }
      C->ipc_state.clear();
      C->ipc_scratch.clear();
    }
  }
  if (C->world > 1 && C->opt.inplace_remap && C->nslots == 1 && !C->d_stage) {
    // receive staging of the in-place exchange: one chunk
    C->stage_bytes = std::min<size_t>(shard_bytes(C), (size_t)256 << 20);
    if (cudaMalloc(&C->d_stage, C->stage_bytes) != cudaSuccess)
      fail(ATLAS_E_OOM, "cudaMalloc(%zu) remap staging failed", C->stage_bytes);
  }
  C->dev_ready = true;
}

template <typename T>
static void upload(void *&d, const std::vector<T> &v) {
  if (d) cudaFree(d);
  d = nullptr;
  size_t b = std::max<size_t>(v.size(), 1) * sizeof(T);
  CK(cudaMalloc(&d, b));
  if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}

static void ensure_blobs(atlas_ctx *C) {
  if (C->blobs_ready) return;
  upload(C->d_coef, C->coef);
  upload(C->d_ops, C->ops);
  upload(C->d_phases, C->phases);
  upload(C->d_mats, C->mats);
  upload(C->d_newpos, C->newpos);
  upload(C->d_ents, C->ents);
  upload(C->d_terms, C->terms);
  C->blobs_ready = true;
}

static void *cur_buf(atlas_ctx *C, int s) { return C->cur[s] ? C->d_scratch[s] : C->d_state[s]; }
static void *other_buf(atlas_ctx *C, int s) { return C->cur[s] ? C->d_state[s] : C->d_scratch[s]; }

// sizes of the simulated ranks' world (virtual mode: slot == rank)
static int slot_rank(const atlas_ctx *C, int s) { return C->nslots > 1 ? s : C->rank; }

std::vector<Xfer> exchange_schedule(const atlas_ctx *C, int k, int r);

// offset at which rank `to` receives the block `from` sends it
static uint64_t recv_offset(const atlas_ctx *C, int k, int from, int to) {
  for (const Xfer &x : exchange_schedule(C, k, to))
    if (x.kind == XFER_RECV && x.peer == from) return x.dst_off;
  fail(ATLAS_E_INVALID, "internal: no receive from %d at %d", from, to);
  return 0;
}

// The exchange of the remap before stage k, for rank r (P:L1312 Shard;
// SURVEY §8e): swapping the g' top local slots with the incoming qubits'
// global slots splits the ranks into groups of 2^g' that differ only in the
// swapped global bits; inside a group every rank sends block b (of 2^g'
// contiguous blocks of its shard) to the rank whose swapped bits are b, where
// it lands at block beta = (sender's swapped bits XOR their flips).
std::vector<Xfer> exchange_schedule(const atlas_ctx *C, int k, int r) {
  const Exchange &ex = C->exch[k];
  const int gp = ex.gp;
  const uint64_t blk = (uint64_t)amp_bytes(C) << (C->L - gp);
  const int nb = 1 << gp;
  u64 Gam = 0;
  for (int j = 0; j < gp; j++) Gam |= 1ull << ex.gamma[j];
  auto dest = [&](int rr, int b, int *rdst, int *beta) {
    int rd = (int)(rr & ~Gam);
    int bt = 0;
    for (int j = 0; j < gp; j++) {
      rd |= ((b >> j) & 1) << ex.gamma[j];
      bt |= (((rr >> ex.gamma[j]) & 1) ^ ex.fI[j]) << j;
    }
    *rdst = rd;
    *beta = bt;
  };
  std::vector<Xfer> v;
  if (gp == 0) return v;
  for (int b = 0; b < nb; b++) {
    int rd, bt;
    dest(r, b, &rd, &bt);
    if (rd == r) v.push_back(Xfer{r, XFER_LOCAL, (uint64_t)b * blk, (uint64_t)bt * blk, blk});
    else v.push_back(Xfer{rd, XFER_SEND, (uint64_t)b * blk, 0, blk});
  }
  int myb = 0;  // the block every peer sends me = my swapped bits
  for (int j = 0; j < gp; j++) myb |= ((r >> ex.gamma[j]) & 1) << j;
  for (int pb = 0; pb < nb; pb++) {
    int p = (int)(r & ~Gam);
    for (int j = 0; j < gp; j++) p |= ((pb >> j) & 1) << ex.gamma[j];
    if (p == r) continue;
    int rd, bt;
    dest(p, myb, &rd, &bt);
    v.push_back(Xfer{p, XFER_RECV, 0, (uint64_t)bt * blk, blk});
  }
  return v;
}

// Fused exchange (option shm_fuse_exchange): the last shared-memory launch
// of stage k-1 stores block b of its packed output (the block the schedule
// sends to rank rd) straight at the offset rank rd receives it at, in rd's
// idle buffer -- a peer's memory over NVLink (CUDA IPC), or another slot's
// buffer in a virtual world.  remote = false: every block to this slot's
// own other buffer (a plain fused pack; the exchange then runs as usual).
static void *rank_other_buf(atlas_ctx *C, int rank) {
  if (C->nslots > 1) return other_buf(C, rank);
  if (rank == C->rank) return other_buf(C, 0);
  return C->cur[0] ? C->ipc_state[rank] : C->ipc_scratch[rank];
}
static bool peer_exchange_ok(const atlas_ctx *C) { return C->nslots > 1 || C->ipc_ready; }
static void fill_peers(atlas_ctx *C, int k, int s, void **peers, bool remote) {
  const int r = slot_rank(C, s);
  const uint64_t blk = (uint64_t)amp_bytes(C) << (C->L - C->exch[k].gp);
  for (const Xfer &x : exchange_schedule(C, k, r)) {
    if (x.kind == XFER_RECV) continue;
    const int b = (int)(x.src_off / blk);
    if (!remote) {
      peers[b] = (char *)other_buf(C, s) + x.src_off;
      continue;
    }
    const uint64_t doff = x.kind == XFER_LOCAL ? x.dst_off : recv_offset(C, k, r, x.peer);
    peers[b] = (char *)rank_other_buf(C, x.peer) + doff;
  }
}

// Exchange of stage k (after the optional pack) for all local slots.
static void do_exchange(atlas_ctx *C, int k) {
  if (C->exch[k].gp == 0) return;
  if (C->nslots > 1) {
    // virtual world: all shards on this device; sends become device copies
    for (int r = 0; r < C->nslots; r++) {
      const char *src = (const char *)cur_buf(C, r);
      for (const Xfer &x : exchange_schedule(C, k, r)) {
        if (x.kind == XFER_RECV) continue;
        char *dst = (char *)other_buf(C, x.peer);
        const uint64_t doff = x.kind == XFER_LOCAL ? x.dst_off : recv_offset(C, k, r, x.peer);
        CK(cudaMemcpyAsync(dst + doff, src + x.src_off, x.bytes, cudaMemcpyDeviceToDevice,
                           C->stream));
      }
    }
    for (int r = 0; r < C->nslots; r++) C->cur[r] ^= 1;
    return;
  }
  if (C->world == 1) return;
  const char *src = (const char *)cur_buf(C, 0);
  char *dst = (char *)other_buf(C, 0);
  NK(g_nccl.groupStart());
  for (const Xfer &x : exchange_schedule(C, k, C->rank)) {
    if (x.kind == XFER_LOCAL)
      CK(cudaMemcpyAsync(dst + x.dst_off, src + x.src_off, x.bytes, cudaMemcpyDeviceToDevice,
                         C->stream));
    else if (x.kind == XFER_SEND)
      NK(g_nccl.send(src + x.src_off, x.bytes, kNcclUint8, x.peer, C->nccl_comm, C->stream));
    else
      NK(g_nccl.recv(dst + x.dst_off, x.bytes, kNcclUint8, x.peer, C->nccl_comm, C->stream));
  }
  NK(g_nccl.groupEnd());
  C->cur[0] ^= 1;
}

// In-place remap (NEXT-3: no second shard buffer at HBM capacity).  The
// pack is a product of bit transpositions (each one in-place pair-swap
// pass); the exchange swaps, for every peer, the block it needs with the
// block it sends -- the schedule of exchange_schedule sends block b to the
// peer whose swapped bits are b and receives that peer's block at
// (its swapped bits ^ incoming flips), i.e. at the SAME offset up to the
// flip relabelling, which one xor-swap pass applies afterwards.
static void pack_inplace(atlas_ctx *C, int s, const int *newpos) {
  const int dt = C->dt == ATLAS_C128 ? 0 : 1;
  const int L = C->L;
  // realise out[newpos(i)] = in[i]: bit j of the input index ends at newpos[j]
  std::vector<int> at(L), who(L);  // at[j]: where input bit j sits now; who[p]: which input bit sits at p
  for (int j = 0; j < L; j++) at[j] = who[j] = j;
  for (int j = 0; j < L; j++) {
    const int t = newpos[j];
    const int p = at[j];
    if (p == t) continue;
    CK(launch_swap_bits(dt, cur_buf(C, s), L, p, t, C->stream));
    const int other = who[t];
    who[t] = j;
    at[j] = t;
    who[p] = other;
    at[other] = p;
  }
}

static void exchange_inplace(atlas_ctx *C, int k) {
  const Exchange &ex = C->exch[k];
  const int gp = ex.gp;
  if (gp == 0) return;
  const int dt = C->dt == ATLAS_C128 ? 0 : 1;
  const size_t B = amp_bytes(C);
  const uint64_t blk = 1ull << (C->L - gp);  // amplitudes per block
  u64 Gam = 0;
  uint64_t f = 0;
  for (int j = 0; j < gp; j++) {
    Gam |= 1ull << ex.gamma[j];
    f |= (uint64_t)ex.fI[j] << j;
  }
  auto bits = [&](int r) {  // swapped bits of rank r
    int b = 0;
    for (int j = 0; j < gp; j++) b |= ((r >> ex.gamma[j]) & 1) << j;
    return b;
  };
  auto peer_of = [&](int r, int d) {  // the rank whose swapped bits are bits(r) ^ d
    int p = r;
    for (int j = 0; j < gp; j++)
      if ((d >> j) & 1) p ^= 1 << ex.gamma[j];
    return p;
  };
  if (C->nslots > 1) {
    for (int r = 0; r < C->nslots; r++)
      for (int d = 1; d < (1 << gp); d++) {
        const int p = peer_of(r, d);
        if (p < r) continue;
        char *a = (char *)cur_buf(C, r) + (uint64_t)bits(p) * blk * B;
        char *b = (char *)cur_buf(C, p) + (uint64_t)bits(r) * blk * B;
        CK(launch_swap_regions(dt, a, b, blk, C->stream));
      }
    for (int r = 0; r < C->nslots; r++)
      CK(launch_xor_swap(dt, cur_buf(C, r), C->L, f << (C->L - gp), C->stream));
    return;
  }
  if (C->world == 1) return;
  // one process per GPU: a perfect matching per step d (every rank pairs
  // with the rank whose swapped bits differ by d), chunked through the
  // staging buffer: send my chunk, receive the peer's into staging, then
  // copy staging over the chunk just sent (stream order)
  char *sh = (char *)cur_buf(C, 0);
  const uint64_t chunk = std::max<uint64_t>(1, C->stage_bytes / B);
  for (int d = 1; d < (1 << gp); d++) {
    const int p = peer_of(C->rank, d);
    char *base = sh + (uint64_t)bits(p) * blk * B;
    for (uint64_t o = 0; o < blk; o += chunk) {
      const uint64_t n = std::min<uint64_t>(chunk, blk - o);
      NK(g_nccl.groupStart());
      NK(g_nccl.send(base + o * B, n * B, kNcclUint8, p, C->nccl_comm, C->stream));
      NK(g_nccl.recv(C->d_stage, n * B, kNcclUint8, p, C->nccl_comm, C->stream));
      NK(g_nccl.groupEnd());
      CK(cudaMemcpyAsync(base + o * B, C->d_stage, n * B, cudaMemcpyDeviceToDevice, C->stream));
    }
  }
  CK(launch_xor_swap(dt, sh, C->L, f << (C->L - gp), C->stream));
}

// Host-DRAM offload tier (NEXT-4; the paper's regional qubits in DRAM,
// Def. P:L1405-1417).  Stage k streams every shard s through
// the GPU: its blocks are gathered from host buffer h_cur by H2D copies
// following stage k's exchange schedule (the all-to-all becomes a choice of
// source addresses), the stage's kernels run, the next remap's pack runs
// (fused into the last shared-memory launch, or standalone), and the shard
// goes back by D2H into the other host buffer.
static void run_offload(atlas_ctx *C) {
  const int dt = C->dt == ATLAS_C128 ? 0 : 1;
  const size_t SB = shard_bytes(C);
  const bool timing = C->opt.timing != 0;
  std::vector<std::pair<int, int64_t>> rec;
  size_t nev = 0;
  auto ev_at = [&](size_t i) {
    while (C->ev.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      C->ev.push_back(e);
    }
    return C->ev[i];
  };
  auto mark = [&](int kind, int64_t bytes) {
    if (!timing) return;
    CK(cudaEventRecord(ev_at(nev++), C->stream));
    rec.push_back({kind, bytes});
  };
  auto mark_end = [&]() {
    if (timing) CK(cudaEventRecord(ev_at(nev++), C->stream));
  };
  const bool from_host = !C->opt.init && C->state_set;
  if (!C->opt.init && !C->state_set) fail(ATLAS_E_ORDER, "option init=0 but no atlas_set_state");
  C->state_set = false;
  C->h_cur = 0;
  const double2 *mats = (const double2 *)C->d_mats;
  const int S = C->sp.s;
  std::vector<size_t> pc(C->nslots, 0);
  for (int k = 0; k < S; k++) {
    char *hsrc = (char *)C->h_buf[C->h_cur];
    char *hdst = (char *)C->h_buf[C->h_cur ^ 1];
    for (int s = 0; s < C->nslots; s++) {
      auto &P = C->prog[s];
      int w = 0;  // device work shard holding the data
      int zm = 0;
      if (k == 0 && !from_host) {
        if (C->opt.init_fuse && !P.empty() && P[0].type == L_SHM && shm_jit_zero_ok(P[0].jit)) {
          zm = s == 0 ? 2 : 1;
        } else {
          mark(L_INIT, (int64_t)SB);
          CK(launch_init(dt, C->d_work[0], C->L, s == 0, C->stream));
          mark_end();
        }
      } else if (k > 0 && C->exch[k].gp > 0) {
        mark(L_H2D, (int64_t)SB);
        for (const Xfer &x : exchange_schedule(C, k, s)) {
          if (x.kind == XFER_SEND) continue;
          uint64_t so = x.src_off;
          const int from = x.kind == XFER_LOCAL ? s : x.peer;
          if (x.kind == XFER_RECV)
            for (const Xfer &y : exchange_schedule(C, k, from))
              if (y.kind == XFER_SEND && y.peer == s) so = y.src_off;
          CK(cudaMemcpyAsync((char *)C->d_work[0] + x.dst_off, hsrc + (size_t)from * SB + so, x.bytes,
                             cudaMemcpyHostToDevice, C->stream));
        }
        mark_end();
      } else {
        mark(L_H2D, (int64_t)SB);
        CK(cudaMemcpyAsync(C->d_work[0], hsrc + (size_t)s * SB, SB, cudaMemcpyHostToDevice, C->stream));
        mark_end();
      }
      // the stage's launches (remap pack / exchange records of stage k were
      // consumed above or at the end of stage k-1)
      while (pc[s] < P.size() && P[pc[s]].stage == k && (P[pc[s]].type == L_PACK || P[pc[s]].type == L_EXCHANGE))
        pc[s]++;
      bool first = true;
      while (pc[s] < P.size() && P[pc[s]].stage == k) {
        const Launch &ln = P[pc[s]++];
        void *st = C->d_work[w];
        const int z = first ? zm : 0;
        first = false;
        mark(ln.type, z ? ln.bytes / 2 : ln.bytes);
        switch (ln.type) {
          case L_FUSED: CK(launch_fused(dt, st, C->L, ln.fl, mats, C->stream)); break;
          case L_SHM: {
            ShmLaunch sl = ln.sl;
            sl.grid_cap = C->opt.shm_grid;
            const bool operm = sl.out_perm_off >= 0;
            void *dst = operm ? C->d_work[w ^ 1] : st;
            if (ln.jit) {
              CK(launch_shm_jit(ln.jit, st, dst, sl, C->stream, z, 0, nullptr, 0));
            } else {
              CK(launch_shm(dt, st, sl, (const ShmOp *)C->d_ops, (const double *)C->d_coef,
                            (const ShmPhase *)C->d_phases, (const DiagEnt *)C->d_ents,
                            (const PermTerm *)C->d_terms, C->stream));
              if (operm)
                CK(launch_permute(dt, st, dst, C->L, &C->newpos[sl.out_perm_off],
                                  (const int *)C->d_newpos + sl.out_perm_off, C->stream));
            }
            if (operm) w ^= 1;
            break;
          }
          case L_SCALE: CK(launch_scale(dt, st, C->L, ln.sre, ln.sim, C->stream)); break;
          default: fail(ATLAS_E_INVALID, "internal: unexpected launch type %d", ln.type);
        }
        mark_end();
      }
      if (zm && first) fail(ATLAS_E_INVALID, "internal: zero-mode slot without a launch");
      // a standalone pack of the next remap runs while the shard is here
      if (k + 1 < S)
        for (size_t q = pc[s]; q < P.size() && P[q].stage == k + 1 && P[q].type == L_PACK; q++) {
          mark(L_PACK, P[q].bytes);
          CK(launch_permute(dt, C->d_work[w], C->d_work[w ^ 1], C->L, &C->newpos[P[q].newpos_off],
                            (const int *)C->d_newpos + P[q].newpos_off, C->stream));
          mark_end();
          w ^= 1;
        }
      mark(L_D2H, (int64_t)SB);
      CK(cudaMemcpyAsync(hdst + (size_t)s * SB, C->d_work[w], SB, cudaMemcpyDeviceToHost, C->stream));
      mark_end();
    }
    C->h_cur ^= 1;
  }
  CK(cudaStreamSynchronize(C->stream));
  C->launch_ms.clear();
  C->launch_kind.clear();
  C->launch_bytes.clear();
  if (timing)
    for (size_t i = 0; i < rec.size(); i++) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, C->ev[2 * i], C->ev[2 * i + 1]));
      C->launch_ms.push_back(ms);
      C->launch_kind.push_back(rec[i].first);
      C->launch_bytes.push_back(rec[i].second);
    }
}

void run(atlas_ctx *C) {
  if (!C->planned) fail(ATLAS_E_ORDER, "atlas_run before atlas_plan");
  ensure_device(C);
  ensure_blobs(C);
  if (!C->jit_ready) {
    const auto t0 = std::chrono::steady_clock::now();
    for (auto &P : C->prog)
      for (auto &ln : P) ln.jit = nullptr;
    if (C->opt.shm_jit) shm_jit_prepare(C);
    C->jit_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    C->jit_ready = true;
  }
  if (C->offload) {
    run_offload(C);
    return;
  }
  const int dt = C->dt == ATLAS_C128 ? 0 : 1;
  const bool timing = C->opt.timing != 0;
  C->launch_ms.clear();
  C->launch_kind.clear();
  C->launch_bytes.clear();
  std::vector<std::pair<int, int64_t>> rec;  // kind, bytes
  size_t nev = 0;
  auto ev_at = [&](size_t i) {
    while (C->ev.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      C->ev.push_back(e);
    }
    return C->ev[i];
  };
  auto mark = [&](int kind, int64_t bytes) {
    if (!timing) return;
    CK(cudaEventRecord(ev_at(nev++), C->stream));
    rec.push_back({kind, bytes});
  };
  // ATLAS_DEBUG_SYNC=1: synchronise after every launch and name the one
  // that fails (debugging aid; not for timing)
  static const bool dbg_sync = getenv("ATLAS_DEBUG_SYNC") != nullptr;
  int nlaunch = 0;
  auto mark_end = [&]() {
    if (timing) CK(cudaEventRecord(ev_at(nev++), C->stream));
    if (dbg_sync) {
      const cudaError_t e = cudaStreamSynchronize(C->stream);
      fprintf(stderr, "atlas debug: launch %d %s\n", nlaunch, cudaGetErrorString(e));
      if (e != cudaSuccess) fail(ATLAS_E_CUDA, "launch %d: %s", nlaunch, cudaGetErrorString(e));
    }
    nlaunch++;
  };
  // init |0...0>: logical 0 -> physical 0 (no flips at stage 0) on rank 0.
  // When the first launch of stage 0 is a plan-specialised shared-memory
  // kernel it synthesises that input itself (zmode) instead of reading a
  // memset shard: one write-only pass fewer.
  std::vector<int> zmode(C->nslots, 0);
  std::vector<char> from_zero(C->nslots, 0);  // this run starts from |0...0> (or zeros) on slot s
  for (int s = 0; s < C->nslots; s++) {
    if (!C->opt.init && C->state_set) continue;
    from_zero[s] = 1;
    C->cur[s] = 0;
    const auto &P = C->prog[s];
    if (C->opt.init_fuse && !P.empty() && P[0].stage == 0 && P[0].type == L_SHM &&
        shm_jit_zero_ok(P[0].jit)) {
      zmode[s] = slot_rank(C, s) == 0 ? 2 : 1;
      continue;
    }
    mark(L_INIT, (int64_t)shard_bytes(C));
    CK(launch_init(dt, cur_buf(C, s), C->L, slot_rank(C, s) == 0, C->stream));
    mark_end();
  }
  if (!C->opt.init && !C->state_set) fail(ATLAS_E_ORDER, "option init=0 but no atlas_set_state");
  C->state_set = false;
  // zero-support tracking (option zero_skip): a run that starts from
  // |0...0> keeps every local slot that no launch has made active yet at 0,
  // so a tile with a 1 on such a slot holds zeros, and an in-place
  // shared-memory launch maps it to zeros (every op is linear and keeps a
  // tile inside itself): those tiles are not visited.  zq[s] = the slots
  // still known zero on slot s (all of them on ranks whose shard starts all
  // zero: every launch there is skipped until the first exchange).  Tracking
  // stops at the first launch it does not model (fused, interpreter, fused
  // pack) and at the first remap.
  const uint64_t lmask = C->L >= 64 ? ~0ull : (1ull << C->L) - 1;
  std::vector<uint64_t> zq(C->nslots, 0);
  std::vector<bool> zall(C->nslots, false);
  if (C->opt.zero_skip)
    for (int s = 0; s < C->nslots; s++)
      if (from_zero[s]) {  // synthesised by the first launch (zmode) or by the init pass
        zq[s] = lmask;
        zall[s] = slot_rank(C, s) != 0;
      }
  // lazy zeros (option zero_lazy): on a slot whose first launch synthesises
  // |0...0> and whose following stage-0 launches are all modelled by the
  // tracking until every local slot has been active, the zeros are never
  // stored: the first launch writes only tile 0, and every later launch
  // takes the elements of the still-zero region (an active slot in zq) as
  // zero in its first gather instead of using what the shard holds there.  The launch that makes zq
  // empty visits every tile and rewrites the whole shard, so the state is
  // complete from there on.  Otherwise the zeros are stored (as above).
  std::vector<char> lazy(C->nslots, 0);
  if (C->opt.zero_skip && C->opt.zero_lazy && !C->opt.shm_tma)
    for (int s = 0; s < C->nslots; s++) {
      if (zmode[s] != 2) continue;
      const auto &P = C->prog[s];
      uint64_t z = lmask;
      for (size_t i = 0; i < P.size() && P[i].stage == 0; i++) {
        const Launch &ln = P[i];
        if (ln.type != L_SHM || !ln.jit || ln.sl.out_perm_off >= 0) break;
        if (i > 0 && !ln.sl.zfill_cap) break;  // compiled without the zero-fill load
        z &= ln.sl.nonactive;
        if (!z) {
          lazy[s] = 1;
          zmode[s] |= 4;
          break;
        }
      }
    }
  const int S = C->sp.s;
  std::vector<size_t> pc(C->nslots, 0);
  std::vector<char> fused_x(S + 1, 0);  // remap k's exchange done by the launches (fused)
  // autotuning (jit.cpp shm_jit_prepare): launches with two pipeline
  // variants run the one not yet timed, between two events
  struct Tune {
    Launch *ln;
    int which;
    cudaEvent_t e0, e1;
  };
  std::vector<Tune> tunes;
  const double2 *mats = (const double2 *)C->d_mats;
  for (int k = 0; k < S; k++) {
    if (k > 0 && C->exch[k].gp > 0 && fused_x[k]) {
      // every slot's last launch of stage k-1 stored its blocks at their
      // destinations: the data is in every rank's other buffer; ranks that
      // are separate processes agree on it with a 4-byte allreduce, which
      // completes only after every rank's stores (stream order)
      for (int s = 0; s < C->nslots; s++) {
        auto &P = C->prog[s];
        while (pc[s] < P.size() && P[pc[s]].stage == k && P[pc[s]].type == L_EXCHANGE) pc[s]++;
      }
      mark(L_EXCHANGE, 0);
      if (C->nslots == 1 && C->world > 1)
        NK(g_nccl.allReduce(C->d_bar, C->d_bar, 1, kNcclInt32, kNcclSum, C->nccl_comm, C->stream));
      mark_end();
      for (int s = 0; s < C->nslots; s++) C->cur[s] ^= 1;
      std::fill(zq.begin(), zq.end(), 0);
      std::fill(zall.begin(), zall.end(), false);
    } else if (k > 0 && C->exch[k].gp > 0) {
      for (int s = 0; s < C->nslots; s++) {
        auto &P = C->prog[s];
        while (pc[s] < P.size() && P[pc[s]].stage == k && P[pc[s]].type == L_PACK) {
          const Launch &ln = P[pc[s]++];
          mark(L_PACK, ln.bytes);
          if (C->opt.inplace_remap) {
            pack_inplace(C, s, &C->newpos[ln.newpos_off]);
          } else {
            CK(launch_permute(dt, cur_buf(C, s), other_buf(C, s), C->L, &C->newpos[ln.newpos_off],
                              (const int *)C->d_newpos + ln.newpos_off, C->stream));
            C->cur[s] ^= 1;
          }
          mark_end();
        }
        if (pc[s] < P.size() && P[pc[s]].stage == k && P[pc[s]].type == L_EXCHANGE) pc[s]++;
      }
      mark(L_EXCHANGE, C->prog[0].empty() ? 0 : (int64_t)((double)shard_bytes(C) * (1.0 - std::ldexp(1.0, -C->exch[k].gp))) * C->nslots);
      if (C->opt.inplace_remap) exchange_inplace(C, k);
      else do_exchange(C, k);
      mark_end();
      std::fill(zq.begin(), zq.end(), 0);
      std::fill(zall.begin(), zall.end(), false);
    }
    for (int s = 0; s < C->nslots; s++) {
      auto &P = C->prog[s];
      while (pc[s] < P.size() && P[pc[s]].stage == k) {
        const Launch &ln = P[pc[s]++];
        void *st = cur_buf(C, s);
        // a launch that synthesises |0...0> only writes the shard
        const int zm = (k == 0 && pc[s] == 1 && ln.type == L_SHM && ln.jit) ? zmode[s] : 0;
        // zero tiles of this launch (see zq above); lazy zeros: the elements
        // to zero-fill (active slots still in zq)
        uint64_t skip = 0;
        const uint64_t zfill = (lazy[s] && !zm) ? zq[s] : 0;
        if (!zm && zq[s]) {
          if (ln.type == L_SHM && ln.jit && ln.sl.out_perm_off < 0) {
            if (zall[s]) continue;  // the whole shard is zero: nothing to do
            skip = zq[s] & ln.sl.nonactive;
          } else {
            zq[s] = 0;
            zall[s] = false;
          }
        }
        if (ln.type == L_SHM && zq[s]) zq[s] &= ln.sl.nonactive;  // active slots may turn nonzero
        if (zm || skip || zfill) {
          // algorithmic bytes of the tiles visited (write-only from |0...0>;
          // lazy zeros: tile 0 only; an fp64 chain launch does not load the
          // elements whose warp (tile bits >= 5) or register part has a
          // still-zero qubit -- jit.cpp issue_load)
          const double vf = std::ldexp(1.0, -__builtin_popcountll(skip));
          int zb = 0;
          if (zfill && C->dt == ATLAS_C128 && ln.sl.zfill_cap)
            for (int t = 5; t < ln.sl.K; t++) zb += (int)((zfill >> ln.sl.act[t]) & 1);
          const double rf = std::ldexp(1.0, -zb);
          int64_t b = (int64_t)((double)ln.bytes * vf * (1.0 + rf) / 2.0);
          if (zm) b = (zm & 4) ? (int64_t)((double)ln.bytes / 2.0 / (double)ln.sl.ntiles) : ln.bytes / 2;
          mark(ln.type, b);
        } else {
          mark(ln.type, ln.bytes);
        }
        switch (ln.type) {
          case L_FUSED: CK(launch_fused(dt, st, C->L, ln.fl, mats, C->stream)); break;
          case L_SHM: {
            ShmLaunch sl = ln.sl;
            sl.grid_cap = C->opt.shm_grid;
            // a fused remap pack writes the permuted output to the other buffer
            const bool operm = sl.out_perm_off >= 0;
            void *dst = operm ? other_buf(C, s) : st;
            // ... and a fused exchange to the destination ranks' buffers
            const bool pex = operm && sl.peer_gp > 0 && ln.jit && peer_exchange_ok(C);
            void *peers[8] = {nullptr};
            if (operm && sl.peer_gp > 0 && ln.jit) fill_peers(C, k + 1, s, peers, pex);
            if (pex) fused_x[k + 1] = 1;
            if (ln.jit && ln.nvar > 1 && !ln.tune_warm) {
              const_cast<Launch &>(ln).tune_warm = true;  // untimed: the first run after the JIT
              CK(launch_shm_jit(ln.jit, st, dst, sl, C->stream, zm, skip, peers, zfill));
            } else if (ln.jit && ln.nvar > 1) {
              int w = 0;
              while (w < ln.nvar - 1 && ln.tune_ms[w] >= 0) w++;
              Tune t{const_cast<Launch *>(&ln), w, nullptr, nullptr};
              CK(cudaEventCreate(&t.e0));
              CK(cudaEventCreate(&t.e1));
              CK(cudaEventRecord(t.e0, C->stream));
              CK(launch_shm_jit(ln.jit_var[w], st, dst, sl, C->stream, zm, skip, peers, zfill));
              CK(cudaEventRecord(t.e1, C->stream));
              tunes.push_back(t);
            } else if (ln.jit) {
              CK(launch_shm_jit(ln.jit, st, dst, sl, C->stream, zm, skip, peers, zfill));
            } else {
              CK(launch_shm(dt, st, sl, (const ShmOp *)C->d_ops, (const double *)C->d_coef,
                            (const ShmPhase *)C->d_phases, (const DiagEnt *)C->d_ents,
                            (const PermTerm *)C->d_terms, C->stream));
              if (operm)  // the interpreter runs in place; the pack follows
                CK(launch_permute(dt, st, dst, C->L, &C->newpos[sl.out_perm_off],
                                  (const int *)C->d_newpos + sl.out_perm_off, C->stream));
            }
            if (operm && !pex) C->cur[s] ^= 1;
            break;
          }
          case L_SCALE: CK(launch_scale(dt, st, C->L, ln.sre, ln.sim, C->stream)); break;
          default: fail(ATLAS_E_INVALID, "internal: unexpected launch type %d", ln.type);
        }
        mark_end();
      }
    }
  }
  if (!C->opt.async || timing || !tunes.empty())
    CK(cudaStreamSynchronize(C->stream));  // async: the caller syncs its stream
  for (Tune &t : tunes) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, t.e0, t.e1));
    cudaEventDestroy(t.e0);
    cudaEventDestroy(t.e1);
    Launch *L = t.ln;
    L->tune_ms[t.which] = ms;
    if (t.which == L->nvar - 1) {  // every variant timed: keep the fastest
      int best = 0;
      for (int v = 1; v < L->nvar; v++)
        if (L->tune_ms[v] < L->tune_ms[best]) best = v;
      L->jit = L->jit_var[best];
      L->nvar = 0;
    }
  }
  if (timing) {
    for (size_t i = 0; i < rec.size(); i++) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, C->ev[2 * i], C->ev[2 * i + 1]));
      C->launch_ms.push_back(ms);
      C->launch_kind.push_back(rec[i].first);
      C->launch_bytes.push_back(rec[i].second);
    }
  }
}

// logical index -> (rank, offset) in the last stage's layout
static void locate(const atlas_ctx *C, int stage, uint64_t x, int *rank, uint64_t *off) {
  const StageMap &mp = C->maps[stage];
  const std::vector<int> &fl = stage == C->sp.s - 1 ? mp.flip_end : mp.flip_begin;
  uint64_t p = 0;
  for (int q = 0; q < C->n; q++) {
    uint64_t b = ((x >> q) & 1) ^ (uint64_t)fl[q];
    p |= b << mp.sigma[q];
  }
  *rank = (int)(p >> C->L);
  *off = p & ((1ull << C->L) - 1);
}

static bool identity_layout(const atlas_ctx *C, int stage, bool end) {
  const StageMap &mp = C->maps[stage];
  const std::vector<int> &fl = end ? mp.flip_end : mp.flip_begin;
  for (int q = 0; q < C->n; q++)
    if (mp.sigma[q] != q || fl[q]) return false;
  return true;
}

// The data of shard s: a device pointer, or (offload tier) a host pointer
// into the pinned buffer that holds the current stage layout.
static char *shard_data(atlas_ctx *C, int s, bool stage0) {
  if (C->offload) return (char *)C->h_buf[stage0 ? 0 : C->h_cur] + (size_t)s * shard_bytes(C);
  return (char *)(stage0 ? C->d_state[s] : cur_buf(C, s));
}

void get_state(atlas_ctx *C, void *host, uint64_t first, uint64_t count) {
  if (!C->planned || !C->dev_ready) fail(ATLAS_E_ORDER, "atlas_get_state before atlas_run");
  if (count == 0) return;
  if (first + count > (1ull << C->n) || first + count < first) fail(ATLAS_E_INVALID, "range out of bounds");
  const size_t B = amp_bytes(C);
  const int last = C->sp.s - 1;
  CK(cudaSetDevice(C->device));
  const cudaMemcpyKind kind = C->offload ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost;
  if (identity_layout(C, last, true)) {
    // physical == logical: contiguous copies per shard
    uint64_t x = first, end = first + count;
    while (x < end) {
      int r = (int)(x >> C->L);
      uint64_t off = x & ((1ull << C->L) - 1);
      uint64_t len = std::min<uint64_t>(end - x, (1ull << C->L) - off);
      int s = C->nslots > 1 ? r : (r == C->rank ? 0 : -1);
      if (s >= 0)
        CK(cudaMemcpyAsync((char *)host + (x - first) * B, shard_data(C, s, false) + off * B, len * B, kind,
                           C->stream));
      x += len;
    }
    if (!C->opt.async) CK(cudaStreamSynchronize(C->stream));  // async: the caller syncs its stream
    return;
  }
  // general layout, few amplitudes (sampled checks at capacity): one small
  // copy per amplitude instead of moving whole shards
  if (!C->offload && count <= 4096 && count * 64 < (1ull << C->L)) {
    for (uint64_t i = 0; i < count; i++) {
      int r;
      uint64_t off;
      locate(C, last, first + i, &r, &off);
      int s = C->nslots > 1 ? r : (r == C->rank ? 0 : -1);
      if (s < 0) continue;
      CK(cudaMemcpyAsync((char *)host + i * B, (const char *)cur_buf(C, s) + off * B, B,
                         cudaMemcpyDeviceToHost, C->stream));
    }
    CK(cudaStreamSynchronize(C->stream));
    return;
  }
  // general layout: the shard(s) on the host, then gather
  std::vector<std::vector<char>> sh(C->offload ? 0 : C->nslots);
  std::vector<const char *> src(C->nslots);
  for (int s = 0; s < C->nslots; s++) {
    if (C->offload) {
      src[s] = shard_data(C, s, false);
      continue;
    }
    sh[s].resize(shard_bytes(C));
    CK(cudaMemcpy(sh[s].data(), cur_buf(C, s), shard_bytes(C), cudaMemcpyDeviceToHost));
    src[s] = sh[s].data();
  }
  for (uint64_t i = 0; i < count; i++) {
    int r;
    uint64_t off;
    locate(C, last, first + i, &r, &off);
    int s = C->nslots > 1 ? r : (r == C->rank ? 0 : -1);
    if (s < 0) continue;
    memcpy((char *)host + i * B, src[s] + off * B, B);
  }
}

void set_state(atlas_ctx *C, const void *host, uint64_t first, uint64_t count) {
  if (!C->planned) fail(ATLAS_E_ORDER, "atlas_set_state before atlas_plan");
  if (first + count > (1ull << C->n) || first + count < first) fail(ATLAS_E_INVALID, "range out of bounds");
  ensure_device(C);
  CK(cudaSetDevice(C->device));
  const size_t B = amp_bytes(C);
  for (int s = 0; s < C->nslots; s++) C->cur[s] = 0;
  const cudaMemcpyKind kind = C->offload ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice;
  if (identity_layout(C, 0, false)) {
    // logical == physical at stage 0: contiguous copies into each shard
    uint64_t x = first, end = first + count;
    while (x < end) {
      int r = (int)(x >> C->L);
      uint64_t off = x & ((1ull << C->L) - 1);
      uint64_t len = std::min<uint64_t>(end - x, (1ull << C->L) - off);
      int s = C->nslots > 1 ? r : (r == C->rank ? 0 : -1);
      if (s >= 0)
        CK(cudaMemcpyAsync(shard_data(C, s, true) + off * B, (const char *)host + (x - first) * B, len * B,
                           kind, C->stream));
      x += len;
    }
    if (!C->opt.async) CK(cudaStreamSynchronize(C->stream));  // async: the caller syncs its stream
    C->state_set = true;
    return;
  }
  // general stage-0 layout: scatter on the host
  std::vector<std::vector<char>> sh(C->offload ? 0 : C->nslots);
  std::vector<char *> dst(C->nslots);
  for (int s = 0; s < C->nslots; s++) {
    if (C->offload) {
      dst[s] = shard_data(C, s, true);
      continue;
    }
    sh[s].resize(shard_bytes(C));
    CK(cudaMemcpy(sh[s].data(), C->d_state[s], shard_bytes(C), cudaMemcpyDeviceToHost));
    dst[s] = sh[s].data();
  }
  for (uint64_t i = 0; i < count; i++) {
    int r;
    uint64_t off;
    locate(C, 0, first + i, &r, &off);
    int s = C->nslots > 1 ? r : (r == C->rank ? 0 : -1);
    if (s < 0) continue;
    memcpy(dst[s] + off * B, (const char *)host + i * B, B);
  }
  if (!C->offload)
    for (int s = 0; s < C->nslots; s++)
      CK(cudaMemcpy(C->d_state[s], sh[s].data(), shard_bytes(C), cudaMemcpyHostToDevice));
  C->state_set = true;
}

void destroy(atlas_ctx *C) {
  if (C->dev_ready) {
    cudaSetDevice(C->device);
    cudaStreamSynchronize(C->stream);
    for (int i = 0; i < 2; i++) {
      if (C->h_buf[i]) cudaFreeHost(C->h_buf[i]);
      if (C->d_work[i]) cudaFree(C->d_work[i]);
    }
    if (!C->bound)
      for (size_t s = 0; s < C->d_state.size(); s++) {
        if (C->d_state[s]) cudaFree(C->d_state[s]);
        if (C->d_scratch[s]) cudaFree(C->d_scratch[s]);
      }
    for (void *p : {C->d_coef, C->d_ops, C->d_phases, C->d_mats, C->d_newpos, C->d_ents, C->d_terms, C->d_stage})
      if (p) cudaFree(p);
    for (auto e : C->ev) cudaEventDestroy(e);
    if (C->ipc_ready) {
      for (int r = 0; r < (int)C->ipc_state.size(); r++)
        if (r != C->rank) {
          cudaIpcCloseMemHandle(C->ipc_state[r]);
          cudaIpcCloseMemHandle(C->ipc_scratch[r]);
        }
      if (C->d_bar) cudaFree(C->d_bar);
    }
    if (C->own_stream) cudaStreamDestroy(C->stream);
    if (C->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy(C->nccl_comm);
  }
  delete C;
}



void nccl_unique_id(void *out) {
  nccl_load();
  NK(g_nccl.getUniqueId(out));
}

}  // namespace atlas
