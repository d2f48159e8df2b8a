// K7: dense bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// the layer compute of the MiCS step with compute (the
// reference has no GEMM, so this is unpinned by it and checked
// against a plain fp32 matmul).
//
//   C[M,N] (+)= A[M,K] · B[K,N]     bf16 operands, fp32 accumulation in TMEM
//
// Either operand may be K-major or MN-major in global memory, which covers the
// three products of a linear layer without transposes (row-major storage):
//   forward  Y  = X · Wᵀ   A = X  (K-major), B = W  (K-major)
//   dgrad    dX = dY · W   A = dY (K-major), B = W  (N-major)
//   wgrad    dW = dYᵀ · X  A = dY (M-major), B = X  (N-major)
//
// Structure: one CTA per SM; CTA pairs are thread-block clusters of 2 running
// tcgen05 with cta_group::2, persistent over 256 x 256 output tiles:
//   warp 0      TMA producer (both CTAs): CTA r loads rows [128r, 128r+128) of A and
//               columns [128r, 128r+128) of B (128B-swizzled boxes) into its own
//               stage of a 6-stage ring (32 KiB per stage: 16 KiB A + 16 KiB B), the
//               bytes counted on the leader's full[s] barrier
//   warp 1      MMA issuer (leader CTA only): one thread issues
//               tcgen05.mma.cta_group::2 M=256 N=256 K=16, reading both CTAs' shared
//               memory; each CTA's TMEM receives its 128 rows x 256 fp32 columns, in one
//               of two accumulators (2 x 256 columns)
//   warps 2..5  epilogue (both CTAs): tcgen05.ld accumulator rows -> registers ->
//               bf16/fp32 -> swizzled shared memory -> TMA store (cp.reduce.async.bulk
//               .add for C +=), overlapping the next tile's MMAs; register stores when
//               C is not TMA-aligned
// Barriers: full[s] (leader: both CTAs' TMA bytes landed), empty[s] (the leader's
// tcgen05.commit multicast to both CTAs, since the peer's producer writes into its
// own stage that the leader's MMAs read), tmem_full[a] (commit, multicast) and
// tmem_empty[a] (leader: one remote arrival per epilogue warp of both CTAs).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <string>

#include "internal.h"

namespace mics {
namespace {

// One CTA pair (cluster of 2, cta_group::2) computes a 256 x 256 tile: CTA r holds
// rows [128r, 128r+128) of A and columns [128r, 128r+128) of B in its shared memory,
// the leader issues M=256 N=256 MMAs that read both halves, and each CTA's TMEM
// receives its 128 rows x 256 columns.  Per SM and k-block: 16 KiB of A + 16 KiB of B.
constexpr int kBM = 128, kBK = 64;
constexpr int kCluster = 2;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KiB: this CTA's 128 rows of A
constexpr int kGemmThreads = 192;
// epilogue staging for TMA stores: per epilogue warp two 32 x 32 chunks (fp32 worst case)
constexpr uint32_t kEpiChunkBytes = 32 * 32 * 4;
constexpr uint32_t kEpiBytes = 4 * 2 * kEpiChunkBytes;  // 32 KiB
// Tile width N of a CTA pair: 256 (a 256 x 128 pair tile halves the MMA work per
// staged A byte and measured slower on every shape); ~192 KiB of stages.
constexpr int kBN = 256;
constexpr uint32_t kBHalfBytes = kBN / kCluster * kBK * 2;  // this CTA's 128 columns of B
constexpr uint32_t kStageBytes = kABytes + kBHalfBytes;
constexpr int kStages = int((192u << 10) / kStageBytes);
constexpr uint32_t kTmemCols = 2 * kBN;  // double-buffered accumulator
constexpr uint32_t kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 /* align */ + 256 /* barriers */;

struct GemmParams {
  void* c;
  uint64_t ldc;
  int M, N, K;
  int c_bf16;   // output element type: 1 bf16, 0 fp32
  int beta;     // 1: C += A·B (fp32 output only)
  int a_mn;     // A is M-major (A(m,k) at a[k*lda + m])
  int b_mn;     // B is N-major (B(n,k) at b[k*ldb + n])
  unsigned long long* probe;  // MICS_GEMM_PROBE: per-CTA stall cycles [8] (debug), else null
  int tma_store;              // 1: epilogue stores through shared memory with TMA (C map valid)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// both CTAs load into their own shared memory; the bytes are counted on the LEADER's barrier
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap* map, uint32_t dst, uint32_t leader_bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_2sm_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), version 1
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// instruction descriptor: fp32 accumulate, bf16 x bf16, M=256 (pair), N=kBN, majors
__device__ __forceinline__ uint32_t idesc_bf16(int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(kBN >> 3) << 17) | (uint32_t((kCluster * kBM) >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// TMA store of a staged 32 x 32 chunk (clipped to the tensor bounds by the hardware);
// `add` reduces into global memory instead (C += chunk, fp32)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1, int add) {
  if (add)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// wait and, when probing, add the cycles spent to *acc
__device__ __forceinline__ void mbar_wait_probe(uint32_t bar, uint32_t parity, unsigned long long* acc) {
  if (!acc) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  *acc += static_cast<unsigned long long>(clock64() - t0);
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
           const __grid_constant__ CUtensorMap tma_c, GemmParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + kStages * kStageBytes;  // [4 warps][2 buffers][32 x 32 chunk]
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  // bars: full[kStages], empty[kStages], tmem_full[2], tmem_empty[2]; then the TMEM base address
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  const uint32_t tfull0 = smem_u32(bars + 2 * kStages), tempty0 = smem_u32(bars + 2 * kStages + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int crank = int(cluster_rank());  // rank inside the pair; CTA 0 leads
  const uint32_t leader = 0;
  constexpr uint16_t kMask = uint16_t((1u << kCluster) - 1);  // both CTAs of the pair
  const long long t_start = P.probe ? clock64() : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, 1);   // leader: its producer's expect_tx (both CTAs' bytes)
      mbar_init(empty0 + 8 * s, 1);  // the leader's MMA commit, multicast to both CTAs
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);                 // the leader's commit, multicast
      mbar_init(tempty0 + 8 * a, 4 * kCluster);     // leader: one arrival per epilogue warp of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 0) {  // the same warp in both CTAs: one pair allocation
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before();
  cluster_sync();  // barriers and TMEM of both CTAs are ready before anything crosses the pair
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // work unit = one 256 x 256 tile per pair; CTA `crank` owns rows m0 + 128*crank
  // (possibly past M: zero-filled loads, masked stores) and loads B columns
  // n0 + 128*crank (possibly past N: zero-filled); tile t = (n-block t / tiles_m,
  // 256-row block t % tiles_m)
  const int tiles_m = (P.M + kCluster * kBM - 1) / (kCluster * kBM), tiles_n = (P.N + kBN - 1) / kBN;
  const int ntiles = tiles_m * tiles_n, nk = (P.K + kBK - 1) / kBK;
  const int cid = blockIdx.x / kCluster, ncl = gridDim.x / kCluster;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const uint32_t leader_full0 = mapa(full0, leader);
      unsigned long long w_empty = 0, *pw = P.probe ? &w_empty : nullptr;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const int m0 = ((t % tiles_m) * kCluster + crank) * kBM;
        const int nb = (t / tiles_m) * kBN + crank * (kBN / kCluster);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait_probe(empty0 + 8 * stage, phase ^ 1, pw);
          const uint32_t lfull = leader_full0 + 8 * stage;
          if (crank == 0) mbar_expect_tx(full0 + 8 * stage, kCluster * kStageBytes);
          const uint32_t sa = smem_u32(smem + stage * kStageBytes), sb = sa + kABytes;
          const int k0 = kb * kBK;
          if (P.a_mn) {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j) tma_load_2d_2sm(&tma_a, sa + j * 8192, lfull, m0 + 64 * j, k0);
          } else {
            tma_load_2d_2sm(&tma_a, sa, lfull, k0, m0);
          }
          if (P.b_mn) {
#pragma unroll
            for (int j = 0; j < kBN / kCluster / 64; ++j)
              tma_load_2d_2sm(&tma_b, sb + j * 8192, lfull, nb + 64 * j, k0);
          } else {
            tma_load_2d_2sm(&tma_b, sb, lfull, k0, nb);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (P.probe) P.probe[blockIdx.x * 8 + 2] = w_empty;
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {  // ---------------- MMA issuer (leader CTA only)
      const uint32_t idesc = idesc_bf16(P.a_mn, P.b_mn);
      // K-major: the 16-element K slice advances 32 B inside the 128 B swizzle row;
      // MN-major: it advances 16 rows of 128 B.  LBO = distance between 64-wide MN blocks.
      const uint32_t a_step = P.a_mn ? 2048u : 32u, b_step = P.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = P.a_mn ? 8192u : 16u, b_lbo = P.b_mn ? 8192u : 16u;
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      unsigned long long w_te = 0, w_full = 0;
      unsigned long long *pte = P.probe ? &w_te : nullptr, *pfu = P.probe ? &w_full : nullptr;
      for (int t = cid; t < ntiles; t += ncl) {
        mbar_wait_probe(tempty0 + 8 * acc, acc_phase ^ 1, pte);
        fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * kBN);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait_probe(full0 + 8 * stage, phase, pfu);
          fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes), sb = sa + kABytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = umma_desc(sa + k * a_step, a_lbo, 1024);
            const uint64_t bd = umma_desc(sb + k * b_step, b_lbo, 1024);
            umma_bf16_2sm(d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit_2sm_mc(empty0 + 8 * stage, kMask);  // frees this stage in both CTAs once read
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm_mc(tfull0 + 8 * acc, kMask);  // both halves of the accumulator complete
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (P.probe) {
        P.probe[blockIdx.x * 8 + 0] = w_te;
        P.probe[blockIdx.x * 8 + 1] = w_full;
      }
    }
  } else {  // ---------------- epilogue: warps 2..5 of both CTAs, TMEM lane quarter = warp % 4
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t leader_tempty0 = mapa(tempty0, leader);
    int acc = 0;
    uint32_t acc_phase = 0;
    unsigned long long w_tf = 0, busy = 0, *ptf = (P.probe && warp == 2 && lane == 0) ? &w_tf : nullptr;
    for (int t = cid; t < ntiles; t += ncl) {
      const int m0 = ((t % tiles_m) * kCluster + crank) * kBM, n0 = (t / tiles_m) * kBN;
      mbar_wait_probe(tfull0 + 8 * acc, acc_phase, ptf);
      const long long tb0 = ptf ? clock64() : 0;
      fence_after();
      const int m = m0 + row;
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kBN + c * 32), v);
        const int n = n0 + c * 32;
        if (P.tma_store) {
          // stage this warp's 32 rows x 32 columns in shared memory in the TMA
          // swizzled layout (16-byte chunk j of row r at j ^ swizzle(r): conflict-free
          // stores), then one lane stores it to global with TMA (bounds clipped)
          if (n >= P.N || m0 >= P.M) continue;  // whole chunk outside C (warp-uniform)
          const int buf = c & 1;
          uint8_t* stg = epi_smem + (uint32_t(q) * 2 + uint32_t(buf)) * kEpiChunkBytes;
          if (c >= 2) {  // the store issued from this buffer two chunks ago has read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
          }
          if (P.c_bf16) {  // 64 B rows, SWIZZLE_64B: chunk j -> j ^ ((row >> 1) & 3)
            uint8_t* row = stg + lane * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 w;
              w.x = pack_bf16(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
              w.y = pack_bf16(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
              w.z = pack_bf16(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
              w.w = pack_bf16(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
              *reinterpret_cast<uint4*>(row + ((j ^ ((lane >> 1) & 3)) * 16)) = w;
            }
          } else {  // 128 B rows, SWIZZLE_128B: chunk j -> j ^ (row & 7)
            uint8_t* row = stg + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) * 16)) =
                  make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
          __syncwarp();
          if (lane == 0) tma_store_2d(&tma_c, smem_u32(stg), n, m0 + q * 32, P.beta);
          continue;
        }
        if (m >= P.M || n >= P.N) continue;
        if (P.c_bf16) {
          uint16_t* out = static_cast<uint16_t*>(P.c) + uint64_t(m) * P.ldc + n;
          if (n + 32 <= P.N && (P.ldc % 8) == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 w;
              w.x = pack_bf16(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
              w.y = pack_bf16(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
              w.z = pack_bf16(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
              w.w = pack_bf16(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
              reinterpret_cast<uint4*>(out)[j] = w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n + j < P.N) {
                const __nv_bfloat16 h = __float2bfloat16_rn(__uint_as_float(v[j]));
                out[j] = *reinterpret_cast<const uint16_t*>(&h);
              }
          }
        } else {
          float* out = static_cast<float*>(P.c) + uint64_t(m) * P.ldc + n;
          if (n + 32 <= P.N && (P.ldc % 4) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 w = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                     __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
              if (P.beta) {
                const float4 o = reinterpret_cast<const float4*>(out)[j];
                w.x += o.x;
                w.y += o.y;
                w.z += o.z;
                w.w += o.w;
              }
              reinterpret_cast<float4*>(out)[j] = w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n + j < P.N) out[j] = __uint_as_float(v[j]) + (P.beta ? out[j] : 0.0f);
          }
        }
      }
      fence_before();
      __syncwarp();
      if (ptf) busy += static_cast<unsigned long long>(clock64() - tb0);
      if (lane == 0) mbar_arrive_cluster(leader_tempty0 + 8 * acc);  // this warp drained its rows
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (ptf) {
      P.probe[blockIdx.x * 8 + 3] = busy;
      P.probe[blockIdx.x * 8 + 5] = w_tf;
    }
    // staged chunks must be read (and the stores complete) before the CTA exits
    if (P.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  cluster_sync();  // no CTA leaves while its pair may still signal or read it
  if (P.probe && threadIdx.x == 0) P.probe[blockIdx.x * 8 + 4] = static_cast<unsigned long long>(clock64() - t_start);
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                 : "memory");
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    MICS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) raise(MICS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// 2-D bf16 map over a row-major [outer, inner] matrix with leading dimension ld
// (elements), box = 64 inner elements (one 128 B swizzle row) x box_outer rows.
CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_outer) {
  if (reinterpret_cast<uintptr_t>(base) % 16 || (ld * 2) % 16)
    raise(MICS_OUT_OF_RANGE, "gemm: operands need 16-byte aligned base and leading dimension (multiple of 8)");
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {64, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(MICS_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

// 2-D map over the output C [M rows, N inner] for the epilogue's TMA stores: 32 x 32
// boxes, 64 B (bf16, SWIZZLE_64B) or 128 B (fp32, SWIZZLE_128B) rows.  Returns false
// when C is not TMA-aligned (the epilogue then stores from registers).
bool make_c_map(CUtensorMap* m, void* c, uint64_t ldc, int M, int N, bool bf16) {
  const uint64_t esz = bf16 ? 2 : 4;
  if (reinterpret_cast<uintptr_t>(c) % 16 || (ldc * esz) % 16) return false;
  const cuuint64_t dims[2] = {uint64_t(N), uint64_t(M)};
  const cuuint64_t strides[1] = {ldc * esz};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c,
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int gemm_grid(int ntiles, int max_sms, int ctas) {
  // the shared-memory opt-in is per device (a multi-device context plans on several)
  static uint64_t ready = 0;
  static int nsm_of[64] = {};
  int dev = 0;
  MICS_CUDA(cudaGetDevice(&dev));
  if (dev >= 64) raise(MICS_CONFIG_ERROR, "device ordinal beyond 63");
  if (!(ready >> dev & 1)) {
    MICS_CUDA(cudaDeviceGetAttribute(&nsm_of[dev], cudaDevAttrMultiProcessorCount, dev));
    MICS_CUDA(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
    ready |= 1ull << dev;
  }
  const int nsm = nsm_of[dev];
  const int sms = max_sms > 0 && max_sms < nsm ? max_sms : nsm;
  const int clusters = sms / ctas > 0 ? sms / ctas : 1;
  return ctas * (ntiles < clusters ? ntiles : clusters);
}

}  // namespace

GemmLaunch plan_gemm(const void* a, uint64_t lda, int a_mn, const void* b, uint64_t ldb, int b_mn, void* c,
                     uint64_t ldc, mics_dtype c_t, int M, int N, int K, int accumulate, int max_sms) {
  if (M <= 0 || N <= 0 || K <= 0) raise(MICS_OUT_OF_RANGE, "gemm: M, N, K must be positive");
  if (c_t != MICS_F32 && c_t != MICS_BF16) raise(MICS_TYPE_MISMATCH, "gemm: output must be f32 or bf16");
  if (accumulate && c_t != MICS_F32) raise(MICS_TYPE_MISMATCH, "gemm: accumulate needs an f32 output");
  if (ldc < uint64_t(N) || lda < uint64_t(a_mn ? M : K) || ldb < uint64_t(b_mn ? N : K))
    raise(MICS_SIZE_MISMATCH, "gemm: leading dimension smaller than the row");
  GemmLaunch g;
  // A(m,k): K-major -> [M rows, K inner]; M-major -> [K rows, M inner]
  g.ma = a_mn ? make_map(a, uint64_t(M), uint64_t(K), lda, 64) : make_map(a, uint64_t(K), uint64_t(M), lda, kBM);
  g.mb = b_mn ? make_map(b, uint64_t(N), uint64_t(K), ldb, 64)
              : make_map(b, uint64_t(K), uint64_t(N), ldb, uint32_t(kBN / kCluster));  // rows per load
  const char* te = std::getenv("MICS_GEMM_TMA_STORE");  // 0: register stores (A/B runs)
  const bool tma_store = !(te && te[0] == '0') && make_c_map(&g.mc, c, ldc, M, N, c_t == MICS_BF16);
  if (!tma_store) g.mc = g.ma;  // unused placeholder
  GemmParams P{c, ldc, M, N, K, c_t == MICS_BF16, accumulate != 0, a_mn != 0, b_mn != 0, nullptr, tma_store};
  static_assert(sizeof(GemmParams) <= sizeof(g.params), "GemmParams fits");
  memcpy(g.params, &P, sizeof(P));
  const int rows = kCluster * kBM;
  g.ntiles = ((M + rows - 1) / rows) * ((N + kBN - 1) / kBN);  // 256 x 256 pair tiles
  g.grid = gemm_grid(g.ntiles, max_sms, kCluster);
  g.flops = 2.0 * double(M) * double(N) * double(K);
  return g;
}

void launch_gemm(cudaStream_t s, const GemmLaunch& g) {
  GemmParams P;
  memcpy(&P, g.params, sizeof(P));
  // MICS_GEMM_PROBE=1 (debugging, synchronous): per-role stall cycles of this launch
  static const bool probe = [] {
    const char* e = std::getenv("MICS_GEMM_PROBE");
    return e && e[0] == '1';
  }();
  static unsigned long long* d_probe = nullptr;
  if (probe) {
    if (!d_probe) MICS_CUDA(cudaMalloc(&d_probe, 1024 * 8 * sizeof(unsigned long long)));
    MICS_CUDA(cudaMemsetAsync(d_probe, 0, 1024 * 8 * sizeof(unsigned long long), s));
    P.probe = d_probe;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(g.grid));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(kCluster);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MICS_CUDA(cudaLaunchKernelEx(&cfg, k_gemm, g.ma, g.mb, g.mc, P));
  if (probe) {
    std::vector<unsigned long long> h(size_t(g.grid) * 8);
    MICS_CUDA(cudaMemcpyAsync(h.data(), d_probe, h.size() * 8, cudaMemcpyDeviceToHost, s));
    MICS_CUDA(cudaStreamSynchronize(s));
    double a[8] = {};
    int nl = 0;
    for (int b = 0; b < g.grid; ++b) {
      for (int k = 0; k < 8; ++k) a[k] += double(h[size_t(b) * 8 + k]);
      nl += (b % 2 == 0);
    }
    std::fprintf(stderr,
                 "[gemm probe] M=%d N=%d K=%d grid=%d tiles=%d: total %.0f cyc/CTA; MMA wait tmem_empty %.0f, "
                 "full %.0f (leaders); producer wait empty %.0f; epilogue busy %.0f, wait tmem_full %.0f\n",
                 P.M, P.N, P.K, g.grid, g.ntiles, a[4] / g.grid, a[0] / nl, a[1] / nl, a[2] / g.grid, a[3] / g.grid,
                 a[5] / g.grid);
  }
}

}  // namespace mics
