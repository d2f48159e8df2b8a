// sm_100a kernels of the MiCS hot path.
//
//  k_hier    — hierarchical all-gather in one launch (K3): stage-1 tiles publish per-tile
//              flags, stage-3 tiles wait for the node peer's flag of the tile they read.
//  k_copy    — pull all-gather engine (K1/K4): 16 B ld.global.nc from local or
//              NVLink-peer memory, one read feeding up to kMaxDst coalesced stores.
//              Replaces all_gather / hierarchical_all_gather / batched_all_gather
//              (collectives.cpp:103-134, :192-306).
//  k_reduce  — pull reduce-scatter engine (K2) with the reference's fold order:
//              fold_{i=0..p-1} in ascending group position starting from position
//              0's value (collectives.cpp:168-181), fused with bf16->fp32 cast, scale
//              and the shard accumulate of two_hop_micro_step (sync_schedule.hpp:137-141).
//  k_adam    — boundary all-reduce's all-gather phase fused with sharded fp32 Adam (K5).
//  k_generate— counter-based synthetic gradients (K6).
//  Cross-GPU ordering: device-side flag barriers (st.release.sys / ld.acquire.sys
//  on IPC-mapped peer memory), no host round trips.
//
// Every data kernel is a grid-stride loop over fixed-size tiles of a descriptor
// table (segments / jobs); grids are sized to a multiple of the SM count.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"

namespace mics {
namespace {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// streaming 16 B load: read-only for the kernel's lifetime, no L1 allocation
// (peer data is never reused; L2 is bypassed for peer apertures anyway).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_plain(const void* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void st_vec(void* p, const uint4& v) { *reinterpret_cast<uint4*>(p) = v; }

// ---------------------------------------------------------------- programmatic dependent launch
// Every data kernel lets its successor be scheduled immediately (its prologue and
// descriptor staging overlap this kernel's tail).  A kernel that consumes its
// predecessor's results waits for it up front; an independent one waits only
// before exiting, which keeps completion in stream order.
// A dependent kernel triggers its successor only once its own wait returned, so at
// most one grid sits waiting behind a running one (triggering first let a whole
// queue of replays become resident and cost 0.6 us per 1 MiB all-gather on 2 GPUs).
// An independent kernel (the step's per-layer gathers) starts copying at once.  A
// fencing one (dep_first 0) has one thread per CTA wait for the predecessor before
// triggering, so its successor cannot start before its predecessor completed: this
// bounds how many gathers are in flight, and so which ones may share a destination
// slot (step.cpp enqueue_gathers).
__device__ __forceinline__ void pdl_begin(const BarrierArg& b) {
  if (b.dep_first == 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (b.dep_first == 2) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
}
__device__ __forceinline__ void pdl_end(const BarrierArg& b) {
  if (b.dep_first != 1) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- barrier
// Pairwise monotone flags: process w's slot on each peer counts the barriers w has
// reached with that peer.  Memory ordering (strict = 0, the default):
//  - entry announces "my inputs are ready"; they were written by kernels that
//    completed before this one started (stream order, or griddepcontrol.wait),
//    so they already sit in this GPU's L2, which is where peer loads are served.
//    The entry signal is a relaxed store.
//  - exit announces "I finished reading your buffers" AND publishes what this
//    launch wrote (peers read it after the barrier without another one: the
//    boundary Adam's bf16 parameters feed the next step's barrier-free gathers,
//    hierarchical phase 1's stage-1 chunks feed the node peers' phase 2).  So every
//    CTA fences its own stores (fence.acq_rel.gpu after __syncthreads, before its
//    ticket), and the last CTA — which has observed every ticket — issues one
//    system-scope fence before its relaxed signals: fence-to-fence synchronisation
//    through the ticket chain, then a release pattern (fence.sys; st.relaxed.sys)
//    towards the peers.  One MEMBAR.GPU per CTA and one MEMBAR.SYS per launch, only
//    for launches that publish (BarrierArg::publish; 2 us of a 1 MiB all-gather).
// The waiter polls relaxed and acquires once, so its L1 holds nothing stale.
// strict = 1 (MICS_BAR_STRICT) adds system fences around every signal (A/B runs).
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// acq_rel fences: MEMBAR.ALL.{GPU,SYS} without the L1 invalidation (CCTL.IVALL) and
// sequential consistency of __threadfence / __threadfence_system (MEMBAR.SC.*); what
// they order is published by a relaxed store the consumer acquires.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ void bar_signal(const BarrierArg& b, uint64_t add) {
  if (b.strict) __threadfence_system();
  for (uint64_t m = b.mask; m; m &= m - 1) {
    const int w = __ffsll(static_cast<long long>(m)) - 1;
    uint64_t* f = b.tab->remote_flag[w];
    const uint64_t v = b.nbar[w] + add;
    if (b.strict) st_release_sys(f, v); else st_relaxed_sys(f, v);
  }
}

__device__ __forceinline__ void bar_wait(const BarrierArg& b, uint64_t add) {
  for (uint64_t m = b.mask; m; m &= m - 1) {
    const int w = __ffsll(static_cast<long long>(m)) - 1;
    const uint64_t* f = b.tab->local_flag[w];
    const uint64_t target = b.nbar[w] + add;
    while (ld_relaxed_sys(f) < target) __nanosleep(32);
    (void)ld_acquire_sys(f);
  }
}

__device__ void bar_entry(const BarrierArg& b) {
  if (b.mask == 0 || !b.entry) return;
  if (threadIdx.x == 0) {
    if (atomicAdd(&b.tickets[0], 1u) == 0) bar_signal(b, 1);  // first CTA: "inputs ready"
    bar_wait(b, 1);
  }
  __syncthreads();
}

__device__ void bar_exit(const BarrierArg& b) {
  if (b.mask == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (b.exit && b.publish) fence_gpu();  // this CTA's stores before its ticket (publication, see above)
    if (b.strict) __threadfence_system();
    const unsigned t = atomicAdd(&b.tickets[1], 1u);
    if (t == gridDim.x - 1) {  // last CTA: every CTA of this GPU finished its accesses
      const uint64_t k = uint64_t(b.entry ? 1 : 0) + uint64_t(b.exit ? 1 : 0);
      if (b.exit) {
        if (b.publish) fence_sys();  // every CTA's fenced stores, seen through the tickets, first
        bar_signal(b, k);
        bar_wait(b, k);
      }
      for (uint64_t m = b.mask; m; m &= m - 1) {
        const int w = __ffsll(static_cast<long long>(m)) - 1;
        b.nbar[w] += k;
      }
      b.tickets[0] = 0;
      b.tickets[1] = 0;
      __threadfence();
    }
  }
}

template <typename T>
__device__ __forceinline__ int find_desc(const T* __restrict__ d, int n, uint32_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------- K1: copy engine
__global__ void __launch_bounds__(kThreads) k_copy(const CopySeg* __restrict__ gsegs, int nseg, uint32_t table_bytes,
                                                   uint32_t ntiles, BarrierArg bar) {
  extern __shared__ __align__(16) unsigned char smem[];
  const bool staged = table_bytes != 0;  // stage the segment table: the per-tile lookup stays on-chip
  if (staged) {
    const uint4* s = reinterpret_cast<const uint4*>(gsegs);
    uint4* d = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < table_bytes / 16; i += kThreads) d[i] = s[i];
  }
  __syncthreads();
  const CopySeg* segs = staged ? reinterpret_cast<const CopySeg*>(smem) : gsegs;
  pdl_begin(bar);
  bar_entry(bar);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // last segment whose group starts at or before `tile`; stripe groups interleave their tiles
    int idx = find_desc(segs, nseg, tile);
    uint32_t rel = tile - segs[idx].tile0;
    const uint32_t k = segs[idx].gsize;
    if (k > 1) {
      idx = idx - int(k) + 1 + int(rel % k);
      rel /= k;
    }
    const CopySeg& s = segs[idx];
    const uint64_t off = uint64_t(rel) * kCopyTile;
    const uint64_t rem = s.bytes - off;
    const uint32_t nb = rem < kCopyTile ? uint32_t(rem) : kCopyTile;
    const uint32_t ndst = s.ndst;
    const uint8_t* src = s.src + off;
    uintptr_t amask = reinterpret_cast<uintptr_t>(src);
#pragma unroll
    for (int d = 0; d < kMaxDst; ++d)
      if (d < int(ndst)) amask |= reinterpret_cast<uintptr_t>(s.dst[d] + off);
    if ((amask & 15) == 0) {
      const uint32_t nv = nb >> 4;
      uint4 v[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) {
        const uint32_t i = threadIdx.x + u * kThreads;
        if (i < nv) v[u] = ld_stream(src + 16ull * i);
      }
#pragma unroll
      for (int d = 0; d < kMaxDst; ++d) {
        if (d >= int(ndst)) break;
        uint8_t* dst = s.dst[d] + off;
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
          const uint32_t i = threadIdx.x + u * kThreads;
          if (i < nv) st_vec(dst + 16ull * i, v[u]);
        }
      }
      for (uint32_t b = nv * 16 + threadIdx.x; b < nb; b += kThreads) {
        const uint8_t x = src[b];
        for (int d = 0; d < int(ndst); ++d) s.dst[d][off + b] = x;
      }
    } else {  // byte-granular chunks (the reference tests' 1/7/9-byte shards)
      for (uint32_t b = threadIdx.x; b < nb; b += kThreads) {
        const uint8_t x = src[b];
        for (int d = 0; d < int(ndst); ++d) s.dst[d][off + b] = x;
      }
    }
  }
  bar_exit(bar);
  pdl_end(bar);
}

// ---------------------------------------------------------------- K3: hierarchical all-gather, one launch
// Loads of data another CTA or GPU stores during this kernel (published by a flag)
// bypass L1 and the non-coherent path: ld.global.cg, served by the owner's L2.
__device__ __forceinline__ uint4 ld_cg(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ uint8_t ld_cg_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return uint8_t(v);
}

// one tile (<= kCopyTile bytes) from src to dst; `coherent`: src is written during this kernel
template <bool kCoherent>
__device__ __forceinline__ void copy_tile(const uint8_t* src, uint8_t* dst, uint32_t nb) {
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const uint32_t nv = nb >> 4;
    uint4 v[kCopyUnroll];
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) {
      const uint32_t i = threadIdx.x + u * kThreads;
      if (i < nv) v[u] = kCoherent ? ld_cg(src + 16ull * i) : ld_stream(src + 16ull * i);
    }
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) {
      const uint32_t i = threadIdx.x + u * kThreads;
      if (i < nv) st_vec(dst + 16ull * i, v[u]);
    }
    for (uint32_t b = nv * 16 + threadIdx.x; b < nb; b += kThreads) dst[b] = kCoherent ? ld_cg_u8(src + b) : src[b];
  } else {  // byte-granular chunks (the reference tests' 1/7/9-byte shards)
    for (uint32_t b = threadIdx.x; b < nb; b += kThreads) dst[b] = kCoherent ? ld_cg_u8(src + b) : src[b];
  }
}

__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// thread 0 after __syncthreads: the CTA's stores of the tile, then the flag (release pattern)
__device__ __forceinline__ void publish_flag(uint64_t* f, uint64_t v, int sys_scope) {
  if (sys_scope) {
    fence_sys();
    st_relaxed_sys(f, v);
  } else {
    fence_gpu();
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
  }
}
// poll relaxed, acquire once (the data loads that follow are ld.global.cg)
__device__ __forceinline__ void wait_flag(const uint64_t* f, uint64_t v, int sys_scope) {
  if (sys_scope) {
    while (ld_relaxed_sys(f) < v) __nanosleep(64);
    (void)ld_acquire_sys(f);
  } else {
    while (ld_relaxed_gpu(f) < v) __nanosleep(64);
    (void)ld_acquire_gpu(f);
  }
}

// Stage 1 and stage 3 of hierarchical all-gathers in one grid (see HierSeg): one layer
// visit (lag-0 stage-3 segments wait for this launch's stage-1 tiles), or, in the
// comm-only step, stage 1 of visit x with stage 3 of visit x-1 (lag 1: their flags were
// published by the previous launch).  PDL: the launch waits for its predecessor before
// anything (the epoch, and in the step the write-after-read order of the gather slots:
// a rank's launch x completes only after each node peer started launch x, i.e.
// finished launch x-1) and lets its successor launch only at its very end — an early
// successor's CTAs could hold SM slots a not-yet-resident CTA of this grid needs to
// publish the flags resident CTAs are waiting for (profiles/r2/hier_pipe_README.md).
// The grid is one resident wave.
__global__ void __launch_bounds__(kThreads, 3) k_hier(const HierSeg* __restrict__ gsegs, int nseg, uint32_t table_bytes,
                                                   uint32_t ntiles, HierArg ha, BarrierArg bar) {
  extern __shared__ __align__(16) unsigned char smem[];
  const bool staged = table_bytes != 0;
  if (staged) {
    const uint4* s = reinterpret_cast<const uint4*>(gsegs);
    uint4* d = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < table_bytes / 16; i += kThreads) d[i] = s[i];
  }
  __syncthreads();
  const HierSeg* segs = staged ? reinterpret_cast<const HierSeg*>(smem) : gsegs;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  bar_entry(bar);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&ha.ctl->epoch) + 1;
  bool peers_done = ha.peer_mask == 0;  // lag-1 sources: the node peers' previous launch completed
  const uint32_t n1 = ha.interleave_n1, n3 = ntiles - n1, mix = n1 < n3 ? n1 : n3;
  for (uint32_t i = blockIdx.x; i < ntiles; i += gridDim.x) {
    uint32_t tile = i;
    if (n1) {  // alternate the two ranges, then the rest of the longer one
      if (i < 2 * mix) tile = (i & 1) ? n1 + (i >> 1) : (i >> 1);
      else tile = n1 > n3 ? i - mix : n1 + i - 2 * mix + mix;
    }
    int idx = find_desc(segs, nseg, tile);
    uint32_t rel = tile - segs[idx].tile0;
    const uint32_t k = segs[idx].gsize;
    if (k > 1) {
      idx = idx - int(k) + 1 + int(rel % k);
      rel /= k;
    }
    const HierSeg& s = segs[idx];
    const uint64_t off = uint64_t(rel) * kCopyTile;
    const uint64_t rem = s.bytes - off;
    const uint32_t nb = rem < kCopyTile ? uint32_t(rem) : kCopyTile;
    if (s.stage == 3) {
      if (s.lag == 0) {  // the node peer's stage-1 tile of this launch must be published first
        if (threadIdx.x == 0) wait_flag(s.flags + rel, epoch, ha.sys_scope);
        __syncthreads();
      } else if (!peers_done) {  // once per CTA: every node peer finished its previous launch
        if (threadIdx.x == 0)
          for (uint64_t m = ha.peer_mask; m; m &= m - 1)
            wait_flag(ha.tab->done[__ffsll(static_cast<long long>(m)) - 1], epoch - 1, ha.sys_scope);
        __syncthreads();
        peers_done = true;
      }
      copy_tile<true>(s.src + off, s.dst + off, nb);
    } else {
      copy_tile<false>(s.src + off, s.dst + off, nb);
      if (ha.tile_flags) {
        __syncthreads();  // every thread's stores of the tile before the publication
        if (threadIdx.x == 0) publish_flag(s.flags + rel, epoch, ha.sys_scope);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_gpu();  // this CTA's stores before its ticket
    if (atomicAdd(&ha.ctl->ticket, 1u) == gridDim.x - 1) {  // last CTA: the launch is done
      ha.ctl->ticket = 0;
      ha.ctl->epoch = epoch;
      if (ha.my_done) publish_flag(ha.my_done, epoch, ha.sys_scope);  // every CTA's stores, via the tickets
      else fence_gpu();
    }
  }
  bar_exit(bar);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- K2: reduce engine
template <typename T> struct Arith;
template <> struct Arith<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
};
template <> struct Arith<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
};
template <> struct Arith<long long> {  // two's-complement wrap, like the reference's int64_t adds
  static __device__ __forceinline__ long long add(long long a, long long b) {
    return static_cast<long long>(static_cast<unsigned long long>(a) + static_cast<unsigned long long>(b));
  }
  static __device__ __forceinline__ long long mul(long long a, long long) { return a; }
};

// element codecs: InT storage -> AccT, 16 B vectors of VEC elements
template <typename In, typename Acc> struct Codec;
template <> struct Codec<float, float> {
  static constexpr int VEC = 4;
  static __device__ __forceinline__ void unpack(const uint4& r, float (&o)[4]) {
    o[0] = __uint_as_float(r.x); o[1] = __uint_as_float(r.y); o[2] = __uint_as_float(r.z); o[3] = __uint_as_float(r.w);
  }
  static __device__ __forceinline__ float one(const void* p, uint64_t e) { return static_cast<const float*>(p)[e]; }
};
template <> struct Codec<uint16_t, float> {  // bf16 -> fp32 is exact
  static constexpr int VEC = 8;
  static __device__ __forceinline__ void unpack(const uint4& r, float (&o)[8]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  static __device__ __forceinline__ float one(const void* p, uint64_t e) {
    return __uint_as_float(uint32_t(static_cast<const uint16_t*>(p)[e]) << 16);
  }
};
template <> struct Codec<double, double> {
  static constexpr int VEC = 2;
  static __device__ __forceinline__ void unpack(const uint4& r, double (&o)[2]) {
    o[0] = __hiloint2double(int(r.y), int(r.x));
    o[1] = __hiloint2double(int(r.w), int(r.z));
  }
  static __device__ __forceinline__ double one(const void* p, uint64_t e) { return static_cast<const double*>(p)[e]; }
};
template <> struct Codec<long long, long long> {
  static constexpr int VEC = 2;
  static __device__ __forceinline__ void unpack(const uint4& r, long long (&o)[2]) {
    o[0] = static_cast<long long>((uint64_t(r.y) << 32) | r.x);
    o[1] = static_cast<long long>((uint64_t(r.w) << 32) | r.z);
  }
  static __device__ __forceinline__ long long one(const void* p, uint64_t e) {
    return static_cast<const long long*>(p)[e];
  }
};

template <typename Acc>
__device__ __forceinline__ Acc finish(Acc a, const Acc* dst, uint64_t e, Acc scale, int use_scale, int mode) {
  if (use_scale) a = Arith<Acc>::mul(a, scale);
  if (mode == MICS_RS_ACCUMULATE) a = Arith<Acc>::add(dst[e], a);
  else if (mode == MICS_RS_ZERO_ACCUM) a = Arith<Acc>::add(Acc(0), a);
  return a;
}

// Loads U vectors per thread from each of up to P sources (all issued before the
// first add, so every source — local HBM and each NVLink peer — is in flight at
// once), then folds them in ascending group position: the reference's order.
template <typename In, typename Acc, int P, int U>
__device__ __forceinline__ void fold_vecs(const uint8_t* const* srcs, uint32_t p, uint64_t e, uint32_t stride,
                                          Acc (&acc)[U][Codec<In, Acc>::VEC]) {
  using C = Codec<In, Acc>;
  constexpr int VEC = C::VEC;
  uint4 raw[P][U];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (i < int(p)) {
      const In* si = reinterpret_cast<const In*>(srcs[i]);
#pragma unroll
      for (int u = 0; u < U; ++u) raw[i][u] = ld_stream(si + e + uint64_t(u) * stride);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) C::unpack(raw[0][u], acc[u]);
#pragma unroll
  for (int i = 1; i < P; ++i) {
    if (i < int(p)) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        Acc x[VEC];
        C::unpack(raw[i][u], x);
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[u][k] = Arith<Acc>::add(acc[u][k], x[k]);
      }
    }
  }
}

// p > 8: sources in batches of 8 (all loads of a batch in flight), folded in order
template <typename In, typename Acc>
__device__ __forceinline__ void fold_vecs_wide(const uint8_t* const* srcs, uint32_t p, uint64_t e,
                                               Acc (&acc)[1][Codec<In, Acc>::VEC]) {
  using C = Codec<In, Acc>;
  constexpr int VEC = C::VEC;
#pragma unroll 1
  for (uint32_t b = 0; b < p; b += 8) {
    uint4 raw[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (b + i < p) raw[i] = ld_stream(reinterpret_cast<const In*>(srcs[b + i]) + e);
    if (b == 0) C::unpack(raw[0], acc[0]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if ((b > 0 || i > 0) && b + i < p) {
        Acc x[VEC];
        C::unpack(raw[i], x);
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[0][k] = Arith<Acc>::add(acc[0][k], x[k]);
      }
    }
  }
}

template <typename Acc, int VEC>
__device__ __forceinline__ void finish_store(Acc* d, const Acc (&acc)[VEC], const uint4 (&prev_raw)[VEC * sizeof(Acc) / 16],
                                             Acc scale, int use_scale, int mode) {
  constexpr int Q = int(VEC * sizeof(Acc) / 16);
  Acc prev[VEC];
  if (mode == MICS_RS_ACCUMULATE) {
#pragma unroll
    for (int q = 0; q < Q; ++q) memcpy(reinterpret_cast<uint8_t*>(prev) + 16 * q, &prev_raw[q], 16);
  }
  Acc out[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    Acc a = acc[k];
    if (use_scale) a = Arith<Acc>::mul(a, scale);
    if (mode == MICS_RS_ACCUMULATE) a = Arith<Acc>::add(prev[k], a);
    else if (mode == MICS_RS_ZERO_ACCUM) a = Arith<Acc>::add(Acc(0), a);
    out[k] = a;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    uint4 r;
    memcpy(&r, reinterpret_cast<const uint8_t*>(out) + 16 * q, 16);
    st_vec(reinterpret_cast<uint8_t*>(d) + 16 * q, r);
  }
}

// U vectors per thread per call, (kRedUnroll / U) calls per tile
template <typename In, typename Acc, int P, int U>
__device__ __forceinline__ void reduce_tile(const uint8_t* const* srcs, uint32_t p, Acc* dst, uint64_t e0,
                                            Acc scale, int use_scale, int mode) {
  constexpr int VEC = Codec<In, Acc>::VEC;
  constexpr int Q = int(VEC * sizeof(Acc) / 16);
  constexpr uint32_t stride = kThreads * VEC;
#pragma unroll 1
  for (int h = 0; h < kRedUnroll; h += U) {
    const uint64_t e = e0 + (uint64_t(h) * kThreads + threadIdx.x) * VEC;
    uint4 prev[U][Q];  // accumulator reads issued together with the source loads
    if (mode == MICS_RS_ACCUMULATE) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < Q; ++q)
          prev[u][q] = ld_plain(reinterpret_cast<const uint8_t*>(dst + e + uint64_t(u) * stride) + 16 * q);
    }
    Acc acc[U][VEC];
    if constexpr (P > 8) fold_vecs_wide<In, Acc>(srcs, p, e, acc);
    else fold_vecs<In, Acc, P, U>(srcs, p, e, stride, acc);
#pragma unroll
    for (int u = 0; u < U; ++u)
      finish_store<Acc, VEC>(dst + e + uint64_t(u) * stride, acc[u], prev[u], scale, use_scale, mode);
  }
}

// PC = source-count class of the launch (2, 4, 8, or 9 = more than 8): each class
// is its own kernel so the common p=2 case keeps a small register footprint.
template <typename In, typename Acc, int PC>
__global__ void __launch_bounds__(kThreads, 2) k_reduce(const RedJob* __restrict__ gjobs, int njobs,
                                                     uint32_t table_bytes, uint32_t ntiles, Acc scale, int use_scale,
                                                     int mode, BarrierArg bar) {
  using C = Codec<In, Acc>;
  constexpr int VEC = C::VEC;
  constexpr uint32_t TILE = kThreads * kRedUnroll * VEC;
  // stage the job table and its source-pointer arrays in shared memory
  extern __shared__ __align__(16) unsigned char smem[];
  const bool staged = table_bytes != 0;
  if (staged) {
    const uint4* s = reinterpret_cast<const uint4*>(gjobs);
    uint4* d = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < table_bytes / 16; i += kThreads) d[i] = s[i];
  }
  __syncthreads();
  const RedJob* jobs = staged ? reinterpret_cast<const RedJob*>(smem) : gjobs;
  pdl_begin(bar);
  bar_entry(bar);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const RedJob& J = jobs[find_desc(jobs, njobs, tile)];
    const uint64_t e0 = uint64_t(tile - J.tile0) * TILE;
    const uint32_t p = J.p;
    const uint8_t* const* srcs =
        staged ? reinterpret_cast<const uint8_t* const*>(smem + (reinterpret_cast<const char*>(J.srcs) -
                                                                 reinterpret_cast<const char*>(gjobs)))
               : J.srcs;
    Acc* dst = reinterpret_cast<Acc*>(J.dst);
    if (J.aligned && e0 + TILE <= J.valid && e0 + TILE <= J.elems) {
      constexpr int U2 = VEC > 4 ? 2 : 4;  // bf16 input widens 8 lanes per vector: fewer vectors in flight
      if constexpr (PC == 2) reduce_tile<In, Acc, 2, U2>(srcs, p, dst, e0, scale, use_scale, mode);
      else if constexpr (PC == 4) reduce_tile<In, Acc, 4, 2>(srcs, p, dst, e0, scale, use_scale, mode);
      else if constexpr (PC == 8) reduce_tile<In, Acc, 8, 1>(srcs, p, dst, e0, scale, use_scale, mode);
      else reduce_tile<In, Acc, 9, 1>(srcs, p, dst, e0, scale, use_scale, mode);
    } else {  // ragged / unaligned / zero-padded tail: element at a time, same fold
      const uint64_t end = (e0 + TILE < J.elems) ? e0 + TILE : J.elems;
      for (uint64_t e = e0 + threadIdx.x; e < end; e += kThreads) {
        Acc a = Acc(0);
        if (e < J.valid) {
          a = C::one(srcs[0], e);
          for (uint32_t i = 1; i < p; ++i) a = Arith<Acc>::add(a, C::one(srcs[i], e));
        }  // else: every position contributes padding zeros; the fold is +0
        dst[e] = finish(a, dst, e, scale, use_scale, mode);
      }
    }
  }
  bar_exit(bar);
  pdl_end(bar);
}

// ---------------------------------------------------------------- K5: AG phase fused with Adam
__device__ __forceinline__ uint16_t f32_to_bf16(float x) {  // RNE, NaN kept quiet (= oracle)
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7fffffffu) > 0x7f800000u) return uint16_t((b >> 16) | 0x40u);
  b += 0x7fffu + ((b >> 16) & 1u);
  return uint16_t(b >> 16);
}

__device__ __forceinline__ void adam_one(float g, float& p, float& m, float& v, const AdamScalars& sc) {
  g = __fmul_rn(g, sc.grad_scale);
  if (sc.wd != 0.0f) g = __fadd_rn(g, __fmul_rn(sc.wd, p));
  m = __fadd_rn(__fmul_rn(sc.b1, m), __fmul_rn(sc.omb1, g));
  v = __fadd_rn(__fmul_rn(sc.b2, v), __fmul_rn(sc.omb2, __fmul_rn(g, g)));
  const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), sc.bc2_sqrt), sc.eps);
  p = __fsub_rn(p, __fmul_rn(sc.step_size, __fdiv_rn(m, denom)));
}

__global__ void __launch_bounds__(kThreads) k_adam(const AdamJob* __restrict__ jobs, int njobs, uint32_t ntiles,
                                                   AdamScalars sc, const DevScalars* __restrict__ dyn,
                                                   BarrierArg bar) {
  pdl_begin(bar);
  // per-step scalars written by the preceding launch: read only after griddepcontrol.wait
  // (pdl_begin with dep_first 1), never while the setter may still be running
  if (dyn) sc = dyn->sc;
  bar_entry(bar);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const AdamJob& J = jobs[find_desc(jobs, njobs, tile)];
    // tiles interleave the rr slices (tile a -> slice a % rr), so every owner's
    // slice is pulled concurrently instead of all GPUs draining owner 0 first
    const uint32_t a = tile - J.tile0, q = a % J.rr;
    const uint64_t s0 = uint64_t(q) * J.sub;
    const uint64_t send = s0 + J.sub < J.elems ? s0 + J.sub : J.elems;
    const uint64_t e0 = s0 + uint64_t(a / J.rr) * kAdamTile;
    if (e0 >= send) continue;
    if (e0 + kAdamTile <= send) {
      // full tile: every load of the tile (the reduced gradient, mostly from NVLink
      // peers, and the local p, m, v) is issued before the first update
      uint4 gr[kAdamUnroll];
      float4 p[kAdamUnroll], m[kAdamUnroll], v[kAdamUnroll];
#pragma unroll
      for (int u = 0; u < kAdamUnroll; ++u) {
        const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * 4;
        gr[u] = ld_stream(J.srcs[uint32_t(e / J.sub)] + e);  // sub % 4 == 0: one owner per vector
        p[u] = *reinterpret_cast<const float4*>(J.param + e);
        m[u] = *reinterpret_cast<const float4*>(J.m + e);
        v[u] = *reinterpret_cast<const float4*>(J.v + e);
      }
#pragma unroll
      for (int u = 0; u < kAdamUnroll; ++u) {
        const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * 4;
        adam_one(__uint_as_float(gr[u].x), p[u].x, m[u].x, v[u].x, sc);
        adam_one(__uint_as_float(gr[u].y), p[u].y, m[u].y, v[u].y, sc);
        adam_one(__uint_as_float(gr[u].z), p[u].z, m[u].z, v[u].z, sc);
        adam_one(__uint_as_float(gr[u].w), p[u].w, m[u].w, v[u].w, sc);
        *reinterpret_cast<float4*>(J.param + e) = p[u];
        *reinterpret_cast<float4*>(J.m + e) = m[u];
        *reinterpret_cast<float4*>(J.v + e) = v[u];
        if (J.pbf16) {
          uint2 pk;
          pk.x = uint32_t(f32_to_bf16(p[u].x)) | (uint32_t(f32_to_bf16(p[u].y)) << 16);
          pk.y = uint32_t(f32_to_bf16(p[u].z)) | (uint32_t(f32_to_bf16(p[u].w)) << 16);
          *reinterpret_cast<uint2*>(J.pbf16 + e) = pk;
        }
        if (J.gout) st_vec(J.gout + e, gr[u]);
      }
      if (J.param2) {  // second replica of the position: same gradient (already in registers)
#pragma unroll
        for (int u = 0; u < kAdamUnroll; ++u) {
          const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * 4;
          p[u] = *reinterpret_cast<const float4*>(J.param2 + e);
          m[u] = *reinterpret_cast<const float4*>(J.m2 + e);
          v[u] = *reinterpret_cast<const float4*>(J.v2 + e);
        }
#pragma unroll
        for (int u = 0; u < kAdamUnroll; ++u) {
          const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * 4;
          adam_one(__uint_as_float(gr[u].x), p[u].x, m[u].x, v[u].x, sc);
          adam_one(__uint_as_float(gr[u].y), p[u].y, m[u].y, v[u].y, sc);
          adam_one(__uint_as_float(gr[u].z), p[u].z, m[u].z, v[u].z, sc);
          adam_one(__uint_as_float(gr[u].w), p[u].w, m[u].w, v[u].w, sc);
          *reinterpret_cast<float4*>(J.param2 + e) = p[u];
          *reinterpret_cast<float4*>(J.m2 + e) = m[u];
          *reinterpret_cast<float4*>(J.v2 + e) = v[u];
          if (J.pbf16_2) {
            uint2 pk;
            pk.x = uint32_t(f32_to_bf16(p[u].x)) | (uint32_t(f32_to_bf16(p[u].y)) << 16);
            pk.y = uint32_t(f32_to_bf16(p[u].z)) | (uint32_t(f32_to_bf16(p[u].w)) << 16);
            *reinterpret_cast<uint2*>(J.pbf16_2 + e) = pk;
          }
        }
      }
      continue;
    }
#pragma unroll 1
    for (int u = 0; u < kAdamUnroll; ++u) {
      const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * 4;
      if (e >= send) continue;
      if (e + 4 <= send) {
        const uint32_t owner = uint32_t(e / J.sub);  // sub % 4 == 0: one owner per vector
        const uint4 gr = ld_stream(J.srcs[owner] + e);
        float4 p = *reinterpret_cast<const float4*>(J.param + e);
        float4 m = *reinterpret_cast<const float4*>(J.m + e);
        float4 v = *reinterpret_cast<const float4*>(J.v + e);
        const float g[4] = {__uint_as_float(gr.x), __uint_as_float(gr.y), __uint_as_float(gr.z),
                            __uint_as_float(gr.w)};
        adam_one(g[0], p.x, m.x, v.x, sc);
        adam_one(g[1], p.y, m.y, v.y, sc);
        adam_one(g[2], p.z, m.z, v.z, sc);
        adam_one(g[3], p.w, m.w, v.w, sc);
        *reinterpret_cast<float4*>(J.param + e) = p;
        *reinterpret_cast<float4*>(J.m + e) = m;
        *reinterpret_cast<float4*>(J.v + e) = v;
        if (J.pbf16) {
          uint2 pk;
          pk.x = uint32_t(f32_to_bf16(p.x)) | (uint32_t(f32_to_bf16(p.y)) << 16);
          pk.y = uint32_t(f32_to_bf16(p.z)) | (uint32_t(f32_to_bf16(p.w)) << 16);
          *reinterpret_cast<uint2*>(J.pbf16 + e) = pk;
        }
        if (J.gout) st_vec(J.gout + e, gr);
        if (J.param2) {
          float4 p2 = *reinterpret_cast<const float4*>(J.param2 + e);
          float4 m2 = *reinterpret_cast<const float4*>(J.m2 + e);
          float4 v2 = *reinterpret_cast<const float4*>(J.v2 + e);
          adam_one(g[0], p2.x, m2.x, v2.x, sc);
          adam_one(g[1], p2.y, m2.y, v2.y, sc);
          adam_one(g[2], p2.z, m2.z, v2.z, sc);
          adam_one(g[3], p2.w, m2.w, v2.w, sc);
          *reinterpret_cast<float4*>(J.param2 + e) = p2;
          *reinterpret_cast<float4*>(J.m2 + e) = m2;
          *reinterpret_cast<float4*>(J.v2 + e) = v2;
          if (J.pbf16_2) {
            uint2 pk;
            pk.x = uint32_t(f32_to_bf16(p2.x)) | (uint32_t(f32_to_bf16(p2.y)) << 16);
            pk.y = uint32_t(f32_to_bf16(p2.z)) | (uint32_t(f32_to_bf16(p2.w)) << 16);
            *reinterpret_cast<uint2*>(J.pbf16_2 + e) = pk;
          }
        }
      } else {
        for (uint64_t x = e; x < send; ++x) {
          const float g = J.srcs[x / J.sub][x];
          float p = J.param[x], m = J.m[x], v = J.v[x];
          adam_one(g, p, m, v, sc);
          J.param[x] = p;
          J.m[x] = m;
          J.v[x] = v;
          if (J.pbf16) J.pbf16[x] = f32_to_bf16(p);
          if (J.gout) J.gout[x] = g;
          if (J.param2) {
            float p2 = J.param2[x], m2 = J.m2[x], v2 = J.v2[x];
            adam_one(g, p2, m2, v2, sc);
            J.param2[x] = p2;
            J.m2[x] = m2;
            J.v2[x] = v2;
            if (J.pbf16_2) J.pbf16_2[x] = f32_to_bf16(p2);
          }
        }
      }
    }
  }
  bar_exit(bar);
  pdl_end(bar);
}

// ---------------------------------------------------------------- K8: fused tail (all ranks local)
template <typename In>
__device__ __forceinline__ void load4(const uint8_t* base, uint64_t e, float (&x)[4]) {
  if constexpr (sizeof(In) == 4) {
    const uint4 r = ld_stream(reinterpret_cast<const float*>(base) + e);
    x[0] = __uint_as_float(r.x);
    x[1] = __uint_as_float(r.y);
    x[2] = __uint_as_float(r.z);
    x[3] = __uint_as_float(r.w);
  } else {  // bf16 -> fp32 is exact
    const uint2 r = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(base) + e);
    x[0] = __uint_as_float(r.x << 16);
    x[1] = __uint_as_float(r.x & 0xffff0000u);
    x[2] = __uint_as_float(r.y << 16);
    x[3] = __uint_as_float(r.y & 0xffff0000u);
  }
}

template <typename In, int R, int P>
__global__ void __launch_bounds__(kThreads, 2) k_tail(const TailJob* __restrict__ jobs, int njobs, uint32_t ntiles,
                                                     AdamScalars sc, const DevScalars* __restrict__ dyn, int zero_accum,
                                                     BarrierArg bar) {
  pdl_begin(bar);
  if (dyn) sc = dyn->sc;  // after griddepcontrol.wait (dep_first 1), as in k_adam
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const TailJob& J = jobs[find_desc(jobs, njobs, tile)];
    const uint64_t e = uint64_t(tile - J.tile0) * kTailTile + uint64_t(threadIdx.x) * 4;
    if (e >= J.elems) continue;  // elems is a multiple of 8: every vector is whole
    // phase 1: every replica's accumulator and gradient sources in flight, then the folds
    float a[R][4], g[R][P][4];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (!zero_accum) {
        const float4 t = *reinterpret_cast<const float4*>(J.acc[q] + e);
        a[q][0] = t.x;
        a[q][1] = t.y;
        a[q][2] = t.z;
        a[q][3] = t.w;
      }
#pragma unroll
      for (int i = 0; i < P; ++i) load4<In>(J.grads[q * kTailMaxP + i], e, g[q][i]);
    }
    float red[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool valid = e + uint64_t(k) < J.valid;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        float f = 0.0f;  // padding: every position contributes zeros, the fold is +0
        if (valid) {
          f = g[q][0][k];
#pragma unroll
          for (int i = 1; i < P; ++i) f = __fadd_rn(f, g[q][i][k]);
        }
        a[q][k] = zero_accum ? __fadd_rn(0.0f, f) : __fadd_rn(a[q][k], f);  // micro-step accumulate
      }
      red[k] = a[0][k];
#pragma unroll
      for (int q = 1; q < R; ++q) red[k] = __fadd_rn(red[k], a[q][k]);  // boundary fold, ascending replica
    }
    // phase 2: Adam on every replica's state (all loads of the replica set in flight)
    float4 pp[R], mm[R], vv[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      pp[q] = *reinterpret_cast<const float4*>(J.prm[q] + e);
      mm[q] = *reinterpret_cast<const float4*>(J.m[q] + e);
      vv[q] = *reinterpret_cast<const float4*>(J.v[q] + e);
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      adam_one(red[0], pp[q].x, mm[q].x, vv[q].x, sc);
      adam_one(red[1], pp[q].y, mm[q].y, vv[q].y, sc);
      adam_one(red[2], pp[q].z, mm[q].z, vv[q].z, sc);
      adam_one(red[3], pp[q].w, mm[q].w, vv[q].w, sc);
      *reinterpret_cast<float4*>(J.prm[q] + e) = pp[q];
      *reinterpret_cast<float4*>(J.m[q] + e) = mm[q];
      *reinterpret_cast<float4*>(J.v[q] + e) = vv[q];
      if (J.bf[q]) {
        uint2 pk;
        pk.x = uint32_t(f32_to_bf16(pp[q].x)) | (uint32_t(f32_to_bf16(pp[q].y)) << 16);
        pk.y = uint32_t(f32_to_bf16(pp[q].z)) | (uint32_t(f32_to_bf16(pp[q].w)) << 16);
        *reinterpret_cast<uint2*>(J.bf[q] + e) = pk;
      }
    }
  }
  pdl_end(bar);
}

// ---------------------------------------------------------------- K6: counter-based gradients
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kThreads) k_generate(void* out, int bf16, uint64_t key, uint64_t start,
                                                       uint64_t count) {
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < count; i += stride) {
    const uint64_t x = splitmix64(key ^ (start + i));
    if (bf16) {
      const float f = float(int32_t(x >> 56) - 128) * (1.0f / 128.0f);
      static_cast<uint16_t*>(out)[i] = uint16_t(__float_as_uint(f) >> 16);
    } else {
      static_cast<float*>(out)[i] = float(int32_t(x >> 40) - (1 << 23)) * (1.0f / 8388608.0f);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_cast_bf16(const float* in, uint16_t* out, uint64_t count) {
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < count; i += stride)
    out[i] = f32_to_bf16(in[i]);
}

// ---------------------------------------------------------------- K9: fused layer-group boundary
__device__ __forceinline__ void adam4(const float4& g, float* prm, float* m, float* v, uint16_t* bf, uint64_t e,
                                      const AdamScalars& sc) {
  float4 p = *reinterpret_cast<const float4*>(prm + e);
  float4 mm = *reinterpret_cast<const float4*>(m + e);
  float4 vv = *reinterpret_cast<const float4*>(v + e);
  adam_one(g.x, p.x, mm.x, vv.x, sc);
  adam_one(g.y, p.y, mm.y, vv.y, sc);
  adam_one(g.z, p.z, mm.z, vv.z, sc);
  adam_one(g.w, p.w, mm.w, vv.w, sc);
  *reinterpret_cast<float4*>(prm + e) = p;
  *reinterpret_cast<float4*>(m + e) = mm;
  *reinterpret_cast<float4*>(v + e) = vv;
  if (bf) {
    uint2 pk;
    pk.x = uint32_t(f32_to_bf16(p.x)) | (uint32_t(f32_to_bf16(p.y)) << 16);
    pk.y = uint32_t(f32_to_bf16(p.z)) | (uint32_t(f32_to_bf16(p.w)) << 16);
    *reinterpret_cast<uint2*>(bf + e) = pk;
  }
}

// UA float4 rows of one replica's state (row u at e + u * kThreads * 4), every load
// issued before the first update, like k_adam's full tile
template <int UA>
__device__ __forceinline__ void adam_rows(const uint4 (&gr)[UA], float* prm, float* m, float* v, uint16_t* bf,
                                          uint64_t e, const AdamScalars& sc) {
  constexpr uint32_t stride = kThreads * 4;
  float4 p[UA], mm[UA], vv[UA];
#pragma unroll
  for (int u = 0; u < UA; ++u) {
    p[u] = *reinterpret_cast<const float4*>(prm + e + u * stride);
    mm[u] = *reinterpret_cast<const float4*>(m + e + u * stride);
    vv[u] = *reinterpret_cast<const float4*>(v + e + u * stride);
  }
#pragma unroll
  for (int u = 0; u < UA; ++u) {
    adam_one(__uint_as_float(gr[u].x), p[u].x, mm[u].x, vv[u].x, sc);
    adam_one(__uint_as_float(gr[u].y), p[u].y, mm[u].y, vv[u].y, sc);
    adam_one(__uint_as_float(gr[u].z), p[u].z, mm[u].z, vv[u].z, sc);
    adam_one(__uint_as_float(gr[u].w), p[u].w, mm[u].w, vv[u].w, sc);
    *reinterpret_cast<float4*>(prm + e + u * stride) = p[u];
    *reinterpret_cast<float4*>(m + e + u * stride) = mm[u];
    *reinterpret_cast<float4*>(v + e + u * stride) = vv[u];
    if (bf) {
      uint2 pk;
      pk.x = uint32_t(f32_to_bf16(p[u].x)) | (uint32_t(f32_to_bf16(p[u].y)) << 16);
      pk.y = uint32_t(f32_to_bf16(p[u].z)) | (uint32_t(f32_to_bf16(p[u].w)) << 16);
      *reinterpret_cast<uint2*>(bf + e + u * stride) = pk;
    }
  }
}

// See FbRsJob / FbAdJob (internal.h).  PDL: waits for its predecessor at entry and lets
// its successor launch only at exit (CTAs spin on flags: nothing may take their slots).
// Items are handed out in order from a ticket counter, so every item of an earlier round
// is taken by a running CTA before any item of a later round: an Adam item waits only on
// fold items of earlier rounds, which never wait.  Each CTA takes exactly one ticket past
// the end, so the launch consumes items + gridDim.x tickets and the last of them resets
// the counter for the next launch.  RC = replica-count class (2, 4, 8): the fold keeps 8
// vectors per thread in flight (RC x U), like k_reduce; Adam 4 rows x 4 streams of 16 B.
template <int RC>
__global__ void __launch_bounds__(kThreads, 2) k_fbnd(FbArg fa, AdamScalars sc, const DevScalars* __restrict__ dyn,
                                                      uint64_t epoch, BarrierArg bar) {
  constexpr int U = 8 / RC;
  constexpr int kFbAdamRows = 4;
  constexpr uint32_t kRow = kThreads * 4;  // fp32 elements of one float4 row
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (dyn) {  // a replayed graph: this step's scalars and flag value
    sc = dyn->sc;
    epoch = dyn->epoch;
  }
  bar_entry(bar);
  const uint32_t r = fa.r, nrs = uint32_t(fa.nrs);
  const uint32_t per_round = nrs + uint32_t(fa.nad) * r;
  __shared__ uint32_t s_item;
  const uint32_t items = fa.items, last = items + gridDim.x - 1;
  for (;;) {
    __syncthreads();  // every thread read the previous item
    if (threadIdx.x == 0) {
      const uint32_t t = atomicAdd(fa.ticket, 1u);
      if (t == last) atomicExch(fa.ticket, 0u);
      s_item = t;
    }
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= items) break;
    const uint32_t round = item / per_round, w = item - round * per_round;
    if (w < nrs) {  // fold of block `round` of a local slice
      const FbRsJob& J = fa.rs[w];
      const uint32_t b = round;
      const uint64_t e0 = uint64_t(b) * fa.blk;
      if (e0 >= J.elems) continue;  // this slice has fewer blocks (or the lag rounds)
      const uint64_t end = e0 + fa.blk < J.elems ? e0 + fa.blk : J.elems;
      const uint8_t* const* srcs = reinterpret_cast<const uint8_t* const*>(J.src);
      uint64_t e = e0;
      // full groups of U rows: all r x U sources in flight, the fold in ascending replica order
      for (; e + uint64_t(U) * kRow <= end; e += uint64_t(U) * kRow) {
        float acc[U][4];
        fold_vecs<float, float, RC, U>(srcs, J.r, e + threadIdx.x * 4, kRow, acc);
#pragma unroll
        for (int u = 0; u < U; ++u)
          *reinterpret_cast<float4*>(J.own + e + threadIdx.x * 4 + u * kRow) =
              make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
      }
      for (uint64_t x = e + threadIdx.x; x < end; x += kThreads) {  // the slice's ragged end
        float a = J.src[0][x];
        for (uint32_t q = 1; q < J.r; ++q) a = __fadd_rn(a, J.src[q][x]);
        J.own[x] = a;
      }
      __syncthreads();  // the block's stores, then one flag into every replica's array
      if (threadIdx.x == 0) {
        if (fa.sys_scope) fence_sys(); else fence_gpu();
        for (uint32_t q = 0; q < J.r; ++q) {
          if (fa.sys_scope) st_relaxed_sys(J.flag[q] + b, epoch);
          else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(J.flag[q] + b), "l"(epoch) : "memory");
        }
      }
    } else {  // Adam of block `round - lag` of owner q's slice
      if (round < fa.lag || round - fa.lag >= fa.nblk) continue;
      const uint32_t a = w - nrs, q = a % r, k = round - fa.lag;  // owners interleaved
      const FbAdJob& J = fa.ad[a / r];
      const uint64_t e0 = uint64_t(q) * J.sub + uint64_t(k) * fa.blk;
      const uint64_t send = (uint64_t(q) + 1) * J.sub < J.elems ? (uint64_t(q) + 1) * J.sub : J.elems;
      if (e0 >= send) continue;  // past the end of owner q's slice
      const uint64_t end = e0 + fa.blk < send ? e0 + fa.blk : send;
      if (threadIdx.x == 0) wait_flag(J.flags + uint64_t(q) * J.fstride + k, epoch, fa.sys_scope);
      __syncthreads();
      const float* g = J.owner[q];
      uint64_t e = e0;
      for (; e + uint64_t(kFbAdamRows) * kRow <= end; e += uint64_t(kFbAdamRows) * kRow) {
        const uint64_t et = e + threadIdx.x * 4;
        uint4 gr[kFbAdamRows];  // L2-coherent: written by the owner during this launch
#pragma unroll
        for (int u = 0; u < kFbAdamRows; ++u) gr[u] = ld_cg(g + et + u * kRow);
        adam_rows<kFbAdamRows>(gr, J.prm, J.m, J.v, J.bf, et, sc);
        if (J.prm2) adam_rows<kFbAdamRows>(gr, J.prm2, J.m2, J.v2, J.bf2, et, sc);
      }
      for (e += threadIdx.x * 4; e < end; e += kRow) {  // the slice's ragged end
        if (e + 4 <= end) {
          const uint4 r4 = ld_cg(g + e);
          const float4 gv = make_float4(__uint_as_float(r4.x), __uint_as_float(r4.y), __uint_as_float(r4.z),
                                        __uint_as_float(r4.w));
          adam4(gv, J.prm, J.m, J.v, J.bf, e, sc);
          if (J.prm2) adam4(gv, J.prm2, J.m2, J.v2, J.bf2, e, sc);
        } else {
          for (uint64_t x = e; x < end; ++x) {
            const float gx = *reinterpret_cast<const volatile float*>(g + x);
            float p = J.prm[x], mm = J.m[x], vv = J.v[x];
            adam_one(gx, p, mm, vv, sc);
            J.prm[x] = p;
            J.m[x] = mm;
            J.v[x] = vv;
            if (J.bf) J.bf[x] = f32_to_bf16(p);
            if (J.prm2) {
              float p2 = J.prm2[x], m2 = J.m2[x], v2 = J.v2[x];
              adam_one(gx, p2, m2, v2, sc);
              J.prm2[x] = p2;
              J.m2[x] = m2;
              J.v2[x] = v2;
              if (J.bf2) J.bf2[x] = f32_to_bf16(p2);
            }
          }
        }
      }
    }
  }
  bar_exit(bar);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void k_set_scalars(DevScalars* dst, DevScalars v) { *dst = v; }

__global__ void k_barrier(BarrierArg bar) {
  pdl_begin(bar);
  bar_entry(bar);
  bar_exit(bar);
  pdl_end(bar);
}

}  // namespace

// ---------------------------------------------------------------- launchers
namespace {
bool pdl_enabled() {  // MICS_PDL=0 launches without programmatic stream serialization (debugging)
  static const bool on = [] {
    const char* e = std::getenv("MICS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... P, typename... A>
void launch_ex(void (*kern)(P...), int grid, int block, size_t smem, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  MICS_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}
}  // namespace

// Resident CTAs per SM of each data kernel (with a full shared-memory table):
// grids are sized to exactly one resident wave, nsm x this.
namespace {
template <typename In, typename Acc>
using ReduceFn = void (*)(const RedJob*, int, uint32_t, uint32_t, Acc, int, int, BarrierArg);

template <typename In, typename Acc>
ReduceFn<In, Acc> reduce_kernel(int pc) {
  switch (pc) {
    case 2: return &k_reduce<In, Acc, 2>;
    case 4: return &k_reduce<In, Acc, 4>;
    case 8: return &k_reduce<In, Acc, 8>;
    default: return &k_reduce<In, Acc, 9>;
  }
}

template <typename In, typename Acc>
int reduce_occupancy(int pc) {
  int n = 0;
  MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reduce_kernel<In, Acc>(pc), kThreads, kSmemTable));
  return n;
}
}  // namespace

int reduce_class(uint32_t max_p) { return max_p <= 2 ? 2 : max_p <= 4 ? 4 : max_p <= 8 ? 8 : 9; }

int resident_ctas(int kind, mics_dtype in_t, int pc) {
  int n = 0;
  switch (kind) {
    case 0:
      MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_copy, kThreads, kSmemTable));
      break;
    case 4:
      MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_hier, kThreads, kSmemTable));
      break;
    case 5: {
      int n2 = 0, n4 = 0;
      MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_fbnd<8>, kThreads, 0));
      MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n4, k_fbnd<4>, kThreads, 0));
      MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n2, k_fbnd<2>, kThreads, 0));
      n = std::min(n, std::min(n2, n4));
      break;
    }
    case 1:
      if (in_t == MICS_BF16) n = reduce_occupancy<uint16_t, float>(pc);
      else if (in_t == MICS_F64) n = reduce_occupancy<double, double>(pc);
      else if (in_t == MICS_I64) n = reduce_occupancy<long long, long long>(pc);
      else n = reduce_occupancy<float, float>(pc);
      break;
    default:
      MICS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_adam, kThreads, 0));
      break;
  }
  return n < 1 ? 1 : n;
}

void launch_copy(cudaStream_t s, const CopySeg* segs, int nseg, uint32_t ntiles, int grid, const BarrierArg& bar) {
  const uint32_t tb = uint64_t(nseg) * sizeof(CopySeg) <= uint64_t(kSmemTable) ? uint32_t(nseg * sizeof(CopySeg)) : 0u;
  launch_ex(k_copy, grid, kThreads, tb, s, segs, nseg, tb, ntiles, bar);
}

void launch_hier(cudaStream_t s, const HierSeg* segs, int nseg, uint32_t ntiles, int grid, const HierArg& ha,
                 const BarrierArg& bar) {
  const uint32_t tb = uint64_t(nseg) * sizeof(HierSeg) <= uint64_t(kSmemTable) ? uint32_t(nseg * sizeof(HierSeg)) : 0u;
  launch_ex(k_hier, grid, kThreads, tb, s, segs, nseg, tb, ntiles, ha, bar);
}

uint32_t reduce_tile_elems(mics_dtype in_t) {
  return uint32_t(kThreads * kRedUnroll) * uint32_t(16 / dtype_size(in_t));
}

void launch_reduce(cudaStream_t s, mics_dtype in_t, mics_dtype acc_t, const RedJob* jobs, int njobs,
                   uint64_t table_bytes, uint32_t max_p, uint32_t ntiles, int grid, double scale, int mode,
                   const BarrierArg& bar) {
  const int use_scale = scale != 1.0;
  const uint32_t tb = table_bytes <= uint64_t(kSmemTable) ? uint32_t(table_bytes) : 0u;  // 0 = read from global
  const int pc = reduce_class(max_p);
  if (in_t == MICS_F32 && acc_t == MICS_F32)
    launch_ex(reduce_kernel<float, float>(pc), grid, kThreads, tb, s, jobs, njobs, tb, ntiles, float(scale),
              use_scale, mode, bar);
  else if (in_t == MICS_BF16 && acc_t == MICS_F32)
    launch_ex(reduce_kernel<uint16_t, float>(pc), grid, kThreads, tb, s, jobs, njobs, tb, ntiles, float(scale),
              use_scale, mode, bar);
  else if (in_t == MICS_F64 && acc_t == MICS_F64)
    launch_ex(reduce_kernel<double, double>(pc), grid, kThreads, tb, s, jobs, njobs, tb, ntiles, scale, use_scale,
              mode, bar);
  else if (in_t == MICS_I64 && acc_t == MICS_I64)
    launch_ex(reduce_kernel<long long, long long>(pc), grid, kThreads, tb, s, jobs, njobs, tb, ntiles, 1LL, 0, mode,
              bar);
  else
    raise(MICS_TYPE_MISMATCH, "unsupported reduce dtype combination");
}

void launch_adam(cudaStream_t s, const AdamJob* jobs, int njobs, uint32_t ntiles, int grid, const AdamScalars& sc,
                 const DevScalars* dyn, const BarrierArg& bar) {
  launch_ex(k_adam, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, bar);
}

bool tail_supported(mics_dtype in_t, int r, int p) {
  return (in_t == MICS_F32 || in_t == MICS_BF16) && ((r == 4 && p == 2) || (r == 2 && p == 4) || (r == 1 && p == 8));
}

void launch_tail(cudaStream_t s, mics_dtype in_t, int r, int p, const TailJob* jobs, int njobs, uint32_t ntiles,
                 int grid, const AdamScalars& sc, const DevScalars* dyn, int zero_accum, const BarrierArg& bar) {
  const bool bf = in_t == MICS_BF16;
  if (r == 4 && p == 2)
    bf ? launch_ex(k_tail<uint16_t, 4, 2>, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, zero_accum, bar)
       : launch_ex(k_tail<float, 4, 2>, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, zero_accum, bar);
  else if (r == 2 && p == 4)
    bf ? launch_ex(k_tail<uint16_t, 2, 4>, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, zero_accum, bar)
       : launch_ex(k_tail<float, 2, 4>, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, zero_accum, bar);
  else if (r == 1 && p == 8)
    bf ? launch_ex(k_tail<uint16_t, 1, 8>, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, zero_accum, bar)
       : launch_ex(k_tail<float, 1, 8>, grid, kThreads, 0, s, jobs, njobs, ntiles, sc, dyn, zero_accum, bar);
  else
    raise(MICS_SHAPE_ERROR, "fused tail: unsupported (replicas, group size)");
}

void launch_set_scalars(cudaStream_t s, DevScalars* dst, const DevScalars& v) {
  k_set_scalars<<<1, 1, 0, s>>>(dst, v);
  MICS_CUDA(cudaGetLastError());
}

void launch_generate(cudaStream_t s, void* out, mics_dtype dtype, uint64_t seed, int rank, int step, int layer,
                     uint64_t start, uint64_t count, int grid) {
  if (count == 0) return;
  const uint64_t key = seed ^ (uint64_t(rank) << 40) ^ (uint64_t(step) << 32) ^ (uint64_t(layer) << 24);
  k_generate<<<grid, kThreads, 0, s>>>(out, dtype == MICS_BF16, key, start, count);
  MICS_CUDA(cudaGetLastError());
}

void launch_cast_bf16(cudaStream_t s, const float* in, uint16_t* out, uint64_t count, int grid) {
  if (count == 0) return;
  k_cast_bf16<<<grid, kThreads, 0, s>>>(in, out, count);
  MICS_CUDA(cudaGetLastError());
}

void launch_fbnd(cudaStream_t s, const FbArg& fa, int grid, const AdamScalars& sc, const DevScalars* dyn,
                 uint64_t epoch, const BarrierArg& bar) {
  auto kern = fa.r <= 2 ? k_fbnd<2> : fa.r <= 4 ? k_fbnd<4> : k_fbnd<8>;
  launch_ex(kern, grid, kThreads, 0, s, fa, sc, dyn, epoch, bar);
}

void launch_barrier(cudaStream_t s, const BarrierArg& bar) {
  launch_ex(k_barrier, 1, 32, 0, s, bar);
}

}  // namespace mics
