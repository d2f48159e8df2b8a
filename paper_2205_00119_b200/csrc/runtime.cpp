// Runtime of libmics: context, symmetric arena, CUDA IPC peer mapping, flag
// barriers, descriptor ring, traffic log.  The B200 counterpart of the
// reference's VirtualRankEngine (collectives.hpp:42-62, collectives.cpp:25-67):
// instead of spawning std::threads per call and copying whole buffers into
// mailbox slots, virtual ranks are (GPU, arena region) pairs and peers pull each
// other's data over NVLink/NVSwitch from IPC-mapped memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

namespace mics {

namespace {
constexpr uint64_t kFlagsBytes = 4096;   // arena head: MICS_MAX_WORLD flag slots (u64), rest reserved
constexpr uint64_t kAlign = 256;
constexpr uint64_t kRingBytes = 16ull << 20;
}  // namespace

[[noreturn]] void raise(mics_status code, const std::string& what) {
  throw Error{code, std::string(mics_status_name(code)) + ": " + what};
}

void cuda_check(cudaError_t e, const char* expr, const char* file, int line) {
  if (e != cudaSuccess)
    raise(MICS_CUDA_ERROR, std::string(cudaGetErrorString(e)) + " in " + expr + " (" + file + ":" +
                               std::to_string(line) + ")");
}

void check_group(const mics_ctx* ctx, const int* ranks, int p) {
  if (p < 0 || p > MICS_MAX_GROUP) raise(MICS_OUT_OF_RANGE, "group size " + std::to_string(p) + " out of range");
  if (p > 0 && !ranks) raise(MICS_OUT_OF_RANGE, "null rank list");
  std::vector<char> seen(size_t(ctx->n), 0);
  for (int i = 0; i < p; ++i) {
    if (ranks[i] < 0 || ranks[i] >= ctx->n)
      raise(MICS_OUT_OF_RANGE, "rank " + std::to_string(ranks[i]) + " outside [0, " + std::to_string(ctx->n) + ")");
    if (seen[size_t(ranks[i])]++) raise(MICS_SHAPE_ERROR, "collective group has duplicate ranks");  // collectives.cpp:19-23
  }
}

AdamScalars make_adam_scalars(double lr, double b1, double b2, double eps, double wd, int step, double grad_scale) {
  // scalars prepared in double then rounded once (the documented Adam formula, include/mics.h)
  AdamScalars s;
  const double bc1 = 1.0 - std::pow(b1, double(step));
  const double bc2 = 1.0 - std::pow(b2, double(step));
  s.b1 = float(b1);
  s.omb1 = float(1.0 - b1);
  s.b2 = float(b2);
  s.omb2 = float(1.0 - b2);
  s.eps = float(eps);
  s.wd = float(wd);
  s.step_size = float(lr / bc1);
  s.bc2_sqrt = float(std::sqrt(bc2));
  s.grad_scale = float(grad_scale);
  return s;
}

}  // namespace mics

using mics::raise;

uint64_t mics_ctx::peer_mask(const int* ranks, int count) const {
  uint64_t mask = 0;
  bool mine = false;
  for (int i = 0; i < count; ++i) {
    const int w = process_of(ranks[i]);
    if (w == wrank) mine = true;
    else mask |= 1ull << w;
  }
  return mine ? mask : 0;
}

uint64_t mics_ctx::local_alloc(uint64_t bytes) {
  if (world != 1 && !member) raise(MICS_CONFIG_ERROR, "host-buffer API needs a single-process context");
  const uint64_t off = used;
  const uint64_t sz = mics::round_up(bytes ? bytes : 1, mics::kAlign);
  if (off + sz > top)
    raise(MICS_INFEASIBLE, "arena exhausted: need " + std::to_string(sz) + " bytes, " + std::to_string(top - off) +
                               " free (raise arena_bytes)");
  used += sz;
  return off;
}

void* mics_ctx::ring_reserve(uint64_t bytes) {
  bytes = mics::round_up(bytes ? bytes : 16, mics::kAlign);
  if (bytes > ring_cap) raise(MICS_OUT_OF_RANGE, "descriptor table larger than the descriptor ring");
  if (ring_head + bytes > ring_cap) {  // wrap: earlier tables may still be in flight
    MICS_CUDA(cudaStreamSynchronize(stream));
    ring_head = 0;
  }
  void* d = ring + ring_head;
  ring_head += bytes;
  return d;
}

void mics_ctx::ring_upload(void* dev, const void* host, uint64_t bytes) {
  // pageable source: the runtime stages it before returning, so `host` may die.
  MICS_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, stream));
}

void* mics_ctx::ring_put(const void* host, uint64_t bytes) {
  void* d = ring_reserve(bytes);
  ring_upload(d, host, bytes);
  return d;
}

// ---------------------------------------------------------------------------
// C-ABI: context
namespace mics {
mics_ctx* create_ctx(const mics_init_args* a) {
  if (!a) raise(MICS_OUT_OF_RANGE, "null init args");
  if (a->n_ranks < 1) raise(MICS_OUT_OF_RANGE, "n_ranks must be >= 1");
  if (a->world < 1 || a->world > MICS_MAX_WORLD) raise(MICS_OUT_OF_RANGE, "world must be in [1, 64]");
  if (a->world_rank < 0 || a->world_rank >= a->world) raise(MICS_OUT_OF_RANGE, "world_rank out of range");
  if (a->n_ranks % a->world) raise(MICS_NON_DIVISIBLE, "world must divide n_ranks (node-major rank placement)");
  auto* c = new mics_ctx();
  try {
    c->n = a->n_ranks;
    c->world = a->world;
    c->wrank = a->world_rank;
    c->per = a->n_ranks / a->world;
    c->device = a->device;
    MICS_CUDA(cudaSetDevice(c->device));
    cudaDeviceProp prop;
    MICS_CUDA(cudaGetDeviceProperties(&prop, c->device));
    if (prop.major != 10)
      raise(MICS_CONFIG_ERROR, std::string("libmics is built for sm_100a (B200); device is ") + prop.name);
    c->nsm = prop.multiProcessorCount;
    c->occ_copy = resident_ctas(0, MICS_F32);
    // Independent back-to-back gathers (the step's per-layer all-gathers): at most
    // three are in flight (step.cpp enqueue_gathers), so each needs several CTAs per
    // SM to stream.  C3 step AG phase at N=4, 1/2/3 CTAs per SM: 2.95/2.64/2.55 ms
    // (profiles/r1/pdl_bound).
    c->occ_copy_indep = std::min(c->occ_copy, 3);
    if (const char* e = std::getenv("MICS_COPY_CTAS_PER_SM"))  // tuning knob
      c->occ_copy_indep = std::max(1, std::min(c->occ_copy, std::atoi(e)));
    if (const char* e = std::getenv("MICS_BAR_STRICT")) c->bar_strict = std::atoi(e) != 0;
    c->occ_adam = resident_ctas(2, MICS_F32);
    // the one-launch hierarchical all-gather must be one resident wave (its stage-3
    // tiles wait for other CTAs' stage-1 tiles): at most its occupancy, 3 like the chain
    c->occ_hier = std::min(resident_ctas(4, MICS_F32), 3);
    c->occ_fbnd = resident_ctas(5, MICS_F32);
    const int classes[4] = {2, 4, 8, 9};
    for (int t = 0; t < 4; ++t)
      for (int k = 0; k < 4; ++k) c->occ_reduce[t][k] = resident_ctas(1, mics_dtype(t), classes[k]);
    MICS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    MICS_CUDA(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
    c->cap = (a->arena_bytes ? a->arena_bytes : (1ull << 30)) + kFlagsBytes;
    c->cap = round_up(c->cap, 2ull << 20);
    c->top = c->cap;
    MICS_CUDA(cudaMalloc(&c->base, c->cap));
    MICS_CUDA(cudaMemset(c->base, 0, kFlagsBytes));
    c->used = kFlagsBytes;
    c->peer_base[c->wrank] = c->base;
    constexpr int K = mics_ctx::kChannels;
    static_assert(K * MICS_MAX_WORLD * sizeof(uint64_t) <= kFlagsBytes, "flag slots of every channel fit");
    static_assert(kDoneOffset >= K * MICS_MAX_WORLD * sizeof(uint64_t) && kDoneOffset + 8 * K <= kFlagsBytes,
                  "done counters after the flag slots, inside the arena head");
    MICS_CUDA(cudaMalloc(&c->d_tab, K * sizeof(PeerTab)));
    {
      PeerTab tab[K];
      std::memset(tab, 0, sizeof(tab));
      for (int ch = 0; ch < K; ++ch) tab[ch].done[c->wrank] = reinterpret_cast<uint64_t*>(c->base + kDoneOffset) + ch;
      MICS_CUDA(cudaMemcpy(c->d_tab, tab, sizeof(tab), cudaMemcpyHostToDevice));
    }
    MICS_CUDA(cudaMalloc(&c->d_nbar, K * sizeof(uint64_t) * MICS_MAX_WORLD));
    MICS_CUDA(cudaMemset(c->d_nbar, 0, K * sizeof(uint64_t) * MICS_MAX_WORLD));
    MICS_CUDA(cudaMalloc(&c->d_tickets, K * 2 * sizeof(unsigned)));
    MICS_CUDA(cudaMemset(c->d_tickets, 0, K * 2 * sizeof(unsigned)));
    MICS_CUDA(cudaMalloc(&c->d_hctl, K * sizeof(HierCtl)));
    MICS_CUDA(cudaMemset(c->d_hctl, 0, K * sizeof(HierCtl)));
    c->ring_cap = kRingBytes;
    MICS_CUDA(cudaMalloc(&c->ring, c->ring_cap));
    MICS_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

void destroy_ctx(mics_ctx* c) {
  if (!c) return;
  if (!c->subs.empty()) {  // a multi-device group: its members own everything
    for (mics_ctx* m : c->subs) destroy_ctx(m);
    delete c;
    return;
  }
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->side_stream) cudaStreamSynchronize(c->side_stream);
  for (int w = 0; w < c->world; ++w)
    if (w != c->wrank && c->peer_base[w] && !c->member) cudaIpcCloseMemHandle(c->peer_base[w]);
  cudaFree(c->ring);
  cudaFree(c->d_tickets);
  cudaFree(c->d_hctl);
  cudaFree(c->d_nbar);
  cudaFree(c->d_tab);
  cudaFree(c->base);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  delete c;
}

void ipc_export(mics_ctx* c, void* handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == MICS_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  MICS_CUDA(cudaIpcGetMemHandle(&h, c->base));
  std::memcpy(handle, &h, sizeof(h));
}

namespace {
// flag tables once every peer_base[] is known (IPC-mapped or peer-accessible UVA)
void connect_peers(mics_ctx* c) {
  PeerTab tab[mics_ctx::kChannels];
  std::memset(tab, 0, sizeof(tab));
  for (int ch = 0; ch < mics_ctx::kChannels; ++ch)
    for (int w = 0; w < c->world; ++w) {
      // channel ch, slot w on our arena is written by process w; slot wrank on process w's arena is ours
      tab[ch].local_flag[w] = reinterpret_cast<uint64_t*>(c->base) + ch * MICS_MAX_WORLD + w;
      tab[ch].remote_flag[w] = reinterpret_cast<uint64_t*>(c->peer_base[w]) + ch * MICS_MAX_WORLD + c->wrank;
      tab[ch].done[w] = reinterpret_cast<uint64_t*>(c->peer_base[w] + kDoneOffset) + ch;
    }
  MICS_CUDA(cudaMemcpy(c->d_tab, tab, sizeof(tab), cudaMemcpyHostToDevice));
  c->ipc_ready = c->world > 1;
}
}  // namespace

void ipc_import(mics_ctx* c, const void* handles) {
  if (c->ipc_ready) raise(MICS_CONFIG_ERROR, "IPC handles already imported");
  if (c->member) raise(MICS_CONFIG_ERROR, "a multi-device context connects its GPUs itself");
  MICS_CUDA(cudaSetDevice(c->device));
  for (int w = 0; w < c->world; ++w) {
    if (w == c->wrank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + size_t(w) * MICS_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    MICS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer_base[w] = static_cast<char*>(p);
  }
  connect_peers(c);
}

// One process, several GPUs: one member context per device (member d = "process" d of
// a world of ndev), peer access between every pair, arenas mapped by UVA pointers.
mics_ctx* create_group(const mics_init_args* a, const int* devices, int ndev) {
  if (!a) raise(MICS_OUT_OF_RANGE, "null init args");
  if (ndev < 1 || ndev > MICS_MAX_WORLD || !devices) raise(MICS_OUT_OF_RANGE, "need 1..64 devices");
  if (a->world != 1 || a->world_rank != 0)
    raise(MICS_CONFIG_ERROR, "a multi-device context is one process (world 1, world_rank 0)");
  if (a->n_ranks < 1 || a->n_ranks % ndev)
    raise(MICS_NON_DIVISIBLE, "the device count must divide n_ranks (node-major rank placement)");
  auto* g = new mics_ctx();
  try {
    g->n = a->n_ranks;
    g->world = ndev;
    g->wrank = 0;
    g->per = a->n_ranks / ndev;
    g->device = devices[0];
    for (int d = 0; d < ndev; ++d) {
      mics_init_args s = *a;
      s.world = ndev;
      s.world_rank = d;
      s.device = devices[d];
      mics_ctx* m = create_ctx(&s);
      m->member = true;
      g->subs.push_back(m);
    }
    for (int x = 0; x < ndev; ++x)
      for (int y = 0; y < ndev; ++y) {
        if (devices[x] == devices[y]) continue;
        int ok = 0;
        MICS_CUDA(cudaDeviceCanAccessPeer(&ok, devices[x], devices[y]));
        if (!ok) raise(MICS_CONFIG_ERROR, "no peer access between GPUs " + std::to_string(devices[x]) + " and " +
                                              std::to_string(devices[y]));
        MICS_CUDA(cudaSetDevice(devices[x]));
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[y], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
        else MICS_CUDA(e);
      }
    for (mics_ctx* m : g->subs) {
      for (int w = 0; w < ndev; ++w) m->peer_base[w] = g->subs[size_t(w)]->base;
      MICS_CUDA(cudaSetDevice(m->device));
      connect_peers(m);
    }
    g->nsm = g->subs[0]->nsm;
    g->stream = g->subs[0]->stream;
    g->ipc_ready = ndev > 1;
  } catch (...) {
    for (mics_ctx* m : g->subs) destroy_ctx(m);
    delete g;
    throw;
  }
  return g;
}

mics_buf alloc_sym(mics_ctx* c, uint64_t bytes_per_rank) {
  mics_buf b;
  b.stride = round_up(bytes_per_rank ? bytes_per_rank : 1, kAlign);
  const uint64_t total = b.stride * uint64_t(c->per);
  if (c->used + total > c->top)
    raise(MICS_INFEASIBLE, "arena exhausted: need " + std::to_string(total) + " bytes, " +
                               std::to_string(c->top - c->used) + " free (raise arena_bytes)");
  b.offset = c->used;
  c->used += total;
  return b;
}

mics_buf hier_flags(mics_ctx* c, uint64_t bytes_per_rank) {
  if (c->hflags.stride >= bytes_per_rank) return c->hflags;
  // SPMD: every process grows at the same call; the old region is simply abandoned
  mics_buf b;
  b.stride = round_up(std::max<uint64_t>(bytes_per_rank, 4096), kAlign);
  const uint64_t total = b.stride * uint64_t(c->per);
  if (c->top < c->used + total)
    raise(MICS_INFEASIBLE, "arena exhausted: hierarchical all-gather flags need " + std::to_string(total) +
                               " bytes (raise arena_bytes)");
  c->top -= total;
  b.offset = c->top;
  MICS_CUDA(cudaMemsetAsync(c->base + b.offset, 0, total, c->stream));
  c->hflags = b;
  return b;
}

void check_buf_rank(const mics_ctx* c, mics_buf b, int rank, uint64_t off, uint64_t bytes) {
  if (rank < 0 || rank >= c->n) raise(MICS_OUT_OF_RANGE, "rank " + std::to_string(rank) + " out of range");
  if (off + bytes > b.stride)
    raise(MICS_OUT_OF_RANGE, "access [" + std::to_string(off) + ", " + std::to_string(off + bytes) +
                                 ") outside the rank's " + std::to_string(b.stride) + "-byte region");
}

void barrier_all(mics_ctx* c) {
  if (c->world == 1) return;
  uint64_t mask = 0;
  for (int w = 0; w < c->world; ++w)
    if (w != c->wrank) mask |= 1ull << w;
  launch_barrier(c->stream, c->barrier(mask, 1, 0));
  c->launches++;
}
}  // namespace mics
