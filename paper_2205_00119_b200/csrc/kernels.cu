// sm_100a kernels of the MiCS hot path.
//
//  k_copy    — pull all-gather engine (K1/K3/K4): 16 B ld.global.nc from local or
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

// ---------------------------------------------------------------- barrier
__device__ void bar_entry(const BarrierArg& b) {
  if (b.mask == 0 || !b.entry) return;
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(&b.tickets[0], 1u);
    if (t == 0) {  // first CTA on this GPU announces "inputs ready"
      __threadfence_system();
      for (uint64_t m = b.mask; m; m &= m - 1) {
        const int w = __ffsll(static_cast<long long>(m)) - 1;
        st_release_sys(b.tab->remote_flag[w], b.nbar[w] + 1);
      }
    }
    for (uint64_t m = b.mask; m; m &= m - 1) {
      const int w = __ffsll(static_cast<long long>(m)) - 1;
      const uint64_t target = b.nbar[w] + 1;
      while (ld_acquire_sys(b.tab->local_flag[w]) < target) __nanosleep(64);
    }
  }
  __syncthreads();
}

__device__ void bar_exit(const BarrierArg& b) {
  if (b.mask == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned t = atomicAdd(&b.tickets[1], 1u);
    if (t == gridDim.x - 1) {  // last CTA: every CTA of this GPU finished its accesses
      __threadfence_system();
      const uint64_t k = uint64_t(b.entry ? 1 : 0) + uint64_t(b.exit ? 1 : 0);
      if (b.exit) {
        for (uint64_t m = b.mask; m; m &= m - 1) {
          const int w = __ffsll(static_cast<long long>(m)) - 1;
          st_release_sys(b.tab->remote_flag[w], b.nbar[w] + k);
        }
        for (uint64_t m = b.mask; m; m &= m - 1) {
          const int w = __ffsll(static_cast<long long>(m)) - 1;
          const uint64_t target = b.nbar[w] + k;
          while (ld_acquire_sys(b.tab->local_flag[w]) < target) __nanosleep(64);
        }
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
__global__ void __launch_bounds__(kThreads) k_copy(const CopySeg* __restrict__ segs, int nseg, uint32_t ntiles,
                                                   BarrierArg bar) {
  bar_entry(bar);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const CopySeg s = segs[find_desc(segs, nseg, tile)];
    const uint64_t off = uint64_t(tile - s.tile0) * kCopyTile;
    const uint64_t rem = s.bytes - off;
    const uint32_t nb = rem < kCopyTile ? uint32_t(rem) : kCopyTile;
    const uint8_t* src = s.src + off;
    uintptr_t amask = reinterpret_cast<uintptr_t>(src);
#pragma unroll
    for (int d = 0; d < kMaxDst; ++d)
      if (d < int(s.ndst)) amask |= reinterpret_cast<uintptr_t>(s.dst[d] + off);
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
        if (d >= int(s.ndst)) break;
        uint8_t* dst = s.dst[d] + off;
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
          const uint32_t i = threadIdx.x + u * kThreads;
          if (i < nv) st_vec(dst + 16ull * i, v[u]);
        }
      }
      for (uint32_t b = nv * 16 + threadIdx.x; b < nb; b += kThreads) {
        const uint8_t x = src[b];
        for (int d = 0; d < int(s.ndst); ++d) s.dst[d][off + b] = x;
      }
    } else {  // byte-granular chunks (the reference tests' 1/7/9-byte shards)
      for (uint32_t b = threadIdx.x; b < nb; b += kThreads) {
        const uint8_t x = src[b];
        for (int d = 0; d < int(s.ndst); ++d) s.dst[d][off + b] = x;
      }
    }
  }
  bar_exit(bar);
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

template <typename In, typename Acc>
__global__ void __launch_bounds__(kThreads) k_reduce(const RedJob* __restrict__ jobs, int njobs, uint32_t ntiles,
                                                     Acc scale, int use_scale, int mode, BarrierArg bar) {
  using C = Codec<In, Acc>;
  constexpr int VEC = C::VEC;
  constexpr uint32_t TILE = kThreads * kRedUnroll * VEC;
  bar_entry(bar);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const RedJob& J = jobs[find_desc(jobs, njobs, tile)];
    const uint64_t e0 = uint64_t(tile - J.tile0) * TILE;
    const uint32_t p = J.p;
    const uint8_t* const* srcs = J.srcs;
    Acc* dst = reinterpret_cast<Acc*>(J.dst);
    if (J.aligned && e0 + TILE <= J.valid && e0 + TILE <= J.elems) {
      Acc acc[kRedUnroll][VEC];
      {
        const In* s0 = reinterpret_cast<const In*>(srcs[0]);
        uint4 raw[kRedUnroll];
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u) raw[u] = ld_stream(s0 + e0 + uint64_t(u * kThreads + threadIdx.x) * VEC);
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u) C::unpack(raw[u], acc[u]);
      }
#pragma unroll 4
      for (uint32_t i = 1; i < p; ++i) {  // ascending group position: the pinned fold order
        const In* si = reinterpret_cast<const In*>(srcs[i]);
        uint4 raw[kRedUnroll];
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u) raw[u] = ld_stream(si + e0 + uint64_t(u * kThreads + threadIdx.x) * VEC);
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u) {
          Acc x[VEC];
          C::unpack(raw[u], x);
#pragma unroll
          for (int k = 0; k < VEC; ++k) acc[u][k] = Arith<Acc>::add(acc[u][k], x[k]);
        }
      }
#pragma unroll
      for (int u = 0; u < kRedUnroll; ++u) {
        const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * VEC;
        Acc* d = dst + e;
        Acc prev[VEC];
        if (mode == MICS_RS_ACCUMULATE) {
#pragma unroll
          for (int q = 0; q < int(VEC * sizeof(Acc) / 16); ++q) {
            const uint4 r = ld_plain(reinterpret_cast<const uint8_t*>(d) + 16 * q);
            memcpy(reinterpret_cast<uint8_t*>(prev) + 16 * q, &r, 16);
          }
        }
        Acc out[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          Acc a = acc[u][k];
          if (use_scale) a = Arith<Acc>::mul(a, scale);
          if (mode == MICS_RS_ACCUMULATE) a = Arith<Acc>::add(prev[k], a);
          else if (mode == MICS_RS_ZERO_ACCUM) a = Arith<Acc>::add(Acc(0), a);
          out[k] = a;
        }
#pragma unroll
        for (int q = 0; q < int(VEC * sizeof(Acc) / 16); ++q) {
          uint4 r;
          memcpy(&r, reinterpret_cast<const uint8_t*>(out) + 16 * q, 16);
          st_vec(reinterpret_cast<uint8_t*>(d) + 16 * q, r);
        }
      }
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
                                                   AdamScalars sc, BarrierArg bar) {
  bar_entry(bar);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const AdamJob& J = jobs[find_desc(jobs, njobs, tile)];
    const uint64_t e0 = uint64_t(tile - J.tile0) * kAdamTile;
#pragma unroll
    for (int u = 0; u < kAdamUnroll; ++u) {
      const uint64_t e = e0 + uint64_t(u * kThreads + threadIdx.x) * 4;
      if (e >= J.elems) continue;
      if (e + 4 <= J.elems) {
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
      } else {
        for (uint64_t x = e; x < J.elems; ++x) {
          const float g = J.srcs[x / J.sub][x];
          float p = J.param[x], m = J.m[x], v = J.v[x];
          adam_one(g, p, m, v, sc);
          J.param[x] = p;
          J.m[x] = m;
          J.v[x] = v;
          if (J.pbf16) J.pbf16[x] = f32_to_bf16(p);
          if (J.gout) J.gout[x] = g;
        }
      }
    }
  }
  bar_exit(bar);
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

__global__ void k_barrier(BarrierArg bar) {
  bar_entry(bar);
  bar_exit(bar);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_copy(cudaStream_t s, const CopySeg* segs, int nseg, uint32_t ntiles, int grid, const BarrierArg& bar) {
  k_copy<<<grid, kThreads, 0, s>>>(segs, nseg, ntiles, bar);
  MICS_CUDA(cudaGetLastError());
}

uint32_t reduce_tile_elems(mics_dtype in_t) {
  return uint32_t(kThreads * kRedUnroll) * uint32_t(16 / dtype_size(in_t));
}

void launch_reduce(cudaStream_t s, mics_dtype in_t, mics_dtype acc_t, const RedJob* jobs, int njobs, uint32_t ntiles,
                   int grid, double scale, int mode, const BarrierArg& bar) {
  const int use_scale = scale != 1.0;
  if (in_t == MICS_F32 && acc_t == MICS_F32)
    k_reduce<float, float><<<grid, kThreads, 0, s>>>(jobs, njobs, ntiles, float(scale), use_scale, mode, bar);
  else if (in_t == MICS_BF16 && acc_t == MICS_F32)
    k_reduce<uint16_t, float><<<grid, kThreads, 0, s>>>(jobs, njobs, ntiles, float(scale), use_scale, mode, bar);
  else if (in_t == MICS_F64 && acc_t == MICS_F64)
    k_reduce<double, double><<<grid, kThreads, 0, s>>>(jobs, njobs, ntiles, scale, use_scale, mode, bar);
  else if (in_t == MICS_I64 && acc_t == MICS_I64)
    k_reduce<long long, long long><<<grid, kThreads, 0, s>>>(jobs, njobs, ntiles, 1, 0, mode, bar);
  else
    raise(MICS_TYPE_MISMATCH, "unsupported reduce dtype combination");
  MICS_CUDA(cudaGetLastError());
}

void launch_adam(cudaStream_t s, const AdamJob* jobs, int njobs, uint32_t ntiles, int grid, const AdamScalars& sc,
                 const BarrierArg& bar) {
  k_adam<<<grid, kThreads, 0, s>>>(jobs, njobs, ntiles, sc, bar);
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

void launch_barrier(cudaStream_t s, const BarrierArg& bar) {
  k_barrier<<<1, 32, 0, s>>>(bar);
  MICS_CUDA(cudaGetLastError());
}

}  // namespace mics
