// Internal declarations of libmics (not part of the C-ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "mics.h"

namespace mics {

// --------------------------------------------------------------------------
// errors: C++ exceptions inside the library, mapped to mics_status at the
// C-ABI edge (capi.cpp) with "<Errc>: detail" messages like sdpsim::raise.
struct Error {
  mics_status code;
  std::string what;
};
[[noreturn]] void raise(mics_status code, const std::string& what);
void cuda_check(cudaError_t e, const char* expr, const char* file, int line);
#define MICS_CUDA(x) ::mics::cuda_check((x), #x, __FILE__, __LINE__)

inline size_t dtype_size(mics_dtype t) {
  switch (t) {
    case MICS_I64: return 8;
    case MICS_F32: return 4;
    case MICS_F64: return 8;
    case MICS_BF16: return 2;
  }
  return 0;
}
inline uint64_t ceil_div(uint64_t a, uint64_t b) { return b ? (a + b - 1) / b : 0; }
inline uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }

// --------------------------------------------------------------------------
// device descriptors (shared by host planners and kernels)
constexpr int kMaxDst = 4;       // destinations written from one source read
constexpr int kThreads = 256;    // threads per CTA for every data kernel
constexpr int kCopyUnroll = 8;   // 16 B vectors in flight per thread per tile
constexpr uint32_t kCopyTile = kThreads * kCopyUnroll * 16;  // 32 KiB
constexpr int kRedUnroll = 4;    // vectors per thread per tile (per source)
constexpr int kAdamUnroll = 4;
constexpr int kSmemTable = 16384;  // descriptor tables up to this size are staged in shared memory

struct CopySeg {              // 64 B
  const uint8_t* src;
  uint8_t* dst[kMaxDst];
  uint64_t bytes;
  uint32_t ndst;
  uint32_t tile0;             // first tile of this segment's stripe group
  uint32_t gsize;             // segments in the stripe group (equal sizes, tiles interleaved)
  uint32_t pad_;
};
static_assert(sizeof(CopySeg) == 64, "CopySeg layout");

// Hierarchical all-gather in ONE launch (K3, collectives.cpp:192-291): stage-1
// segments (the channel all-gather among the q ranks sharing a local index, stage 2's
// rearrangement folded into the store address) publish one flag per kCopyTile tile
// once its bytes are stored; stage-3 segments (a node peer's stage-1 chunk, pulled
// into this rank's output) wait for the flag of the tile they read.  All stage-1
// tiles precede all stage-3 tiles in tile order, so a CTA never waits before its own
// stage-1 tiles are done; flags hold the launch's epoch (monotone per channel).
struct HierSeg {              // 64 B
  const uint8_t* src;
  uint8_t* dst;
  uint64_t* flags;            // stage 1: the flags this chunk publishes; stage 3: its source chunk's flags
  uint64_t bytes;
  uint32_t tile0;             // first tile of this segment's stripe group
  uint32_t gsize;             // segments in the stripe group (equal sizes, tiles interleaved)
  uint32_t stage;             // 1 or 3
  uint32_t lag;               // stage 3: its source tiles were published `lag` launches back (0 or 1)
  uint32_t pad_[4];
};
static_assert(sizeof(HierSeg) == 64, "HierSeg layout");
struct HierCtl {              // per barrier channel, device memory
  uint64_t epoch;             // epoch of the last completed k_hier launch
  unsigned ticket;            // CTA arrivals of the running launch
  unsigned pad_;
};
struct PeerTab;
struct HierArg {
  HierCtl* ctl;
  const PeerTab* tab;         // done counters of the peers (channel's table)
  uint64_t* my_done;          // this process's done counter (merged launches), or null
  uint64_t peer_mask;         // lag-1 stage-3 tiles wait until these processes' done >= epoch - 1
  int sys_scope;              // flags / counters read across GPUs
  int tile_flags;             // stage-1 tiles publish per-tile flags (lag-0 stage-3 readers)
  // merged launches: tiles [0, n1) (stage 1) and [n1, ntiles) (stage 3 of the previous
  // visit) are taken alternately, so NVLink pulls and HBM copies run side by side all
  // through the launch (0 = in order: lag-0 stage-3 tiles must follow every stage-1 tile)
  uint32_t interleave_n1;
};

struct RedJob {               // one output chunk (one destination rank, one segment)
  const uint8_t* const* srcs; // p source pointers, already offset to this chunk
  uint8_t* dst;
  uint64_t elems;             // chunk elements
  uint64_t valid;             // elements [valid, elems) read as zero
  uint32_t p;
  uint32_t tile0;
  uint32_t aligned;           // all srcs and dst 16-byte aligned
  uint32_t pad_;
};

struct AdamJob {              // boundary: all-gather phase fused with Adam, one local rank
  const float* const* srcs;   // rr shard base pointers (replication positions)
  float* param;
  float* m;
  float* v;
  uint16_t* pbf16;            // nullable
  float* gout;                // nullable: write the reduced gradient back
  uint64_t elems;
  uint64_t sub;               // slice owned by each replication position (multiple of 4)
  uint32_t rr;
  uint32_t tile0;
  // optional second local replica of the same position (same reduced gradient, its own
  // state): the gradient is pulled once and both replicas are updated (nullable)
  float* param2;
  float* m2;
  float* v2;
  uint16_t* pbf16_2;
};

struct AdamScalars {
  float b1, omb1, b2, omb2, eps, wd, step_size, bc2_sqrt, grad_scale;
};

// Per-step values of a replayed (CUDA-graph) step, read by the boundary kernels
// from device memory instead of their by-value parameters: the Adam scalars
// (bias correction changes every step).
struct DevScalars {
  AdamScalars sc;
  uint32_t pad_;
  uint64_t epoch;  // the fused layer-group boundaries' flag value of this step (K9)
};

// Fused tail (K8, every rank on this GPU): the last micro-step's reduce-scatter, the
// boundary all-reduce and Adam in one pass over (partition position j, layer): for
// every replica q of position j, a_q = acc_q (+)= fold_i grads_{q,i}; red = fold_q a_q;
// Adam on replica q's state with red.  Same operations in the same order as the
// K2 + K2 + K5 sequence it replaces, without writing / re-reading a_q and red.
constexpr int kTailMaxR = 8, kTailMaxP = 8;
constexpr uint32_t kTailTile = kThreads * 4;  // fp32 elements per tile (one float4 per thread)
struct TailJob {
  const float* acc[kTailMaxR];                    // replica q's accumulator (shard, this layer)
  const uint8_t* grads[kTailMaxR * kTailMaxP];   // [q][i]: member i of replica q's group, chunk j
  float* prm[kTailMaxR];
  float* m[kTailMaxR];
  float* v[kTailMaxR];
  uint16_t* bf[kTailMaxR];                        // nullable
  uint64_t elems, valid;                          // chunk elements (multiple of 8); valid gradient prefix
  uint32_t tile0, pad_;
};

// K9 (`k_fbnd`): the boundary of one layer group in ONE launch, in the overlapped tail of
// multi-process jobs.  Reduce-scatter items: block k of a local rank's slice, `blk`
// elements (fold over the r replicas in ascending order, stored in place), then published
// by a flag pushed into every replica's flag array.  Adam items: block k of owner q's
// slice of a local rank's range, after waiting for owner q's flag of block k.  Items run
// in rounds: round t = the reduce-scatter items of block t, then the Adam items of block
// t - lag (every owner), so NVLink pulls (the fold) and HBM traffic (Adam's state)
// overlap all through the launch.  An Adam item waits only on reduce-scatter items of an
// earlier round, which never wait, and items are taken in order from a ticket counter,
// so every awaited flag is produced by a running CTA.
uint32_t fb_block();                  // elements per published block (MICS_FB_BLOCK, default 16 Ki)
struct FbRsJob {                      // one local rank's slice of the group
  const float* src[kTailMaxR];        // replica q's shard at this slice
  float* own;                         // this rank's shard at this slice (reduced in place)
  uint64_t* flag[kTailMaxR];          // replica q's flag for this slice's block 0
  uint64_t elems;
  uint32_t r, pad_;
};
struct FbAdJob {                      // one local rank (+ an optional second replica of its position)
  const float* owner[kTailMaxR];      // replica q's shard at the group start (q reduced slice q)
  const uint64_t* flags;              // this rank's flags for the group: owner q, block k at q * fstride + k
  float* prm;
  float* m;
  float* v;
  uint16_t* bf;
  float* prm2;                        // nullable: the second local replica
  float* m2;
  float* v2;
  uint16_t* bf2;
  uint64_t elems, sub;                // group elements; slice length (multiple of the block)
  uint32_t fstride, pad_;             // flags per owner (the largest group's blocks per slice)
};
struct FbArg {                        // one k_fbnd launch (device pointers into its descriptor blob)
  const FbRsJob* rs = nullptr;
  const FbAdJob* ad = nullptr;
  int nrs = 0, nad = 0;
  uint32_t r = 2, nblk = 0, blk = 0, lag = 0;  // replicas; blocks per slice, elements per block; rounds
  uint32_t items = 0;
  uint32_t* ticket = nullptr;         // this GPU's item counter (zero between launches)
  int sys_scope = 0;
};

// Flag barrier between processes: remote_flag[w] is the slot on process w's
// arena reserved for this process; local_flag[w] is the slot process w writes
// on ours.  Values are monotone barrier counts per process pair.
struct PeerTab {
  uint64_t* remote_flag[MICS_MAX_WORLD];
  uint64_t* local_flag[MICS_MAX_WORLD];
  // process w's epoch of its last completed merged k_hier launch on this channel
  // (arena head, kDoneOffset + 8 * channel); self included
  uint64_t* done[MICS_MAX_WORLD];
};
constexpr uint64_t kDoneOffset = 2048;  // arena head: done counters, after the barrier flag slots

struct BarrierArg {
  const PeerTab* tab;
  uint64_t* nbar;             // [MICS_MAX_WORLD] barriers completed with each peer (device, local)
  unsigned* tickets;          // [2] CTA arrival tickets (entry, exit)
  uint64_t mask;              // peers taking part (bit w = process w), never includes self
  int entry;                  // signal + wait before any data access
  int exit;                   // last CTA signals + waits after all data access
  // Programmatic dependent launch: 1 = griddepcontrol.wait before touching memory
  // (the kernel consumes its predecessor's results); 0 and 2 = independent of the
  // predecessor (barrier-free all-gathers of static shards): it waits only at its
  // end, so completion order — and every transitive dependency — is preserved.
  // 0 ("fence") lets its successor start only once its own predecessor completed;
  // 2 lets it start at once.  A chain with a fence every m gathers therefore has at
  // most m+1 consecutive gathers in flight (step.cpp enqueue_gathers).
  int dep_first;
  // 1 = full system fences around every signal (the conservative protocol, kept
  // for A/B runs: MICS_BAR_STRICT=1); 0 = relaxed signals, see bar_entry/bar_exit
  int strict;
  // 1 = the exit barrier also publishes this launch's stores to the peers (a fence per
  // CTA + one system fence, kernels.cu bar_exit): set where a peer reads what this
  // launch wrote without an entry barrier of its own in between (all-reduce's
  // reduce-scatter phase, hierarchical phase 1, the boundary's reduce-scatter and Adam).
  // 0 for launches whose outputs are only read by later launches that enter through
  // their own barrier (plain all-gather / reduce-scatter, the micro-step reduce-scatter).
  int publish = 1;
};

// --------------------------------------------------------------------------
// kernel launchers (kernels.cu)
void launch_copy(cudaStream_t s, const CopySeg* segs, int nseg, uint32_t ntiles, int grid, const BarrierArg& bar);
void launch_hier(cudaStream_t s, const HierSeg* segs, int nseg, uint32_t ntiles, int grid, const HierArg& ha,
                 const BarrierArg& bar);
// `table_bytes`: size of the uploaded job table + source-pointer arrays (staged in smem when small)
void launch_reduce(cudaStream_t s, mics_dtype in_t, mics_dtype acc_t, const RedJob* jobs, int njobs,
                   uint64_t table_bytes, uint32_t max_p, uint32_t ntiles, int grid, double scale, int mode,
                   const BarrierArg& bar);
uint32_t reduce_tile_elems(mics_dtype in_t);
int reduce_class(uint32_t max_p);  // 2, 4, 8 or 9 (> 8 sources)
int resident_ctas(int kind /* 0 copy, 1 reduce, 2 adam, 4 hier, 5 fused boundary */, mics_dtype in_t,
                  int pclass = 2);
void launch_adam(cudaStream_t s, const AdamJob* jobs, int njobs, uint32_t ntiles, int grid, const AdamScalars& sc,
                 const DevScalars* dyn, const BarrierArg& bar);
void launch_set_scalars(cudaStream_t s, DevScalars* dst, const DevScalars& v);
// false when (r, p) has no instantiation (the caller keeps the unfused tail)
bool tail_supported(mics_dtype in_t, int r, int p);
void launch_tail(cudaStream_t s, mics_dtype in_t, int r, int p, const TailJob* jobs, int njobs, uint32_t ntiles,
                 int grid, const AdamScalars& sc, const DevScalars* dyn, int zero_accum, const BarrierArg& bar);
constexpr uint32_t kAdamTile = kThreads * kAdamUnroll * 4;
void launch_generate(cudaStream_t s, void* out, mics_dtype dtype, uint64_t seed, int rank, int step, int layer,
                     uint64_t start, uint64_t count, int grid);
void launch_cast_bf16(cudaStream_t s, const float* in, uint16_t* out, uint64_t count, int grid);
void launch_barrier(cudaStream_t s, const BarrierArg& bar);
void launch_fbnd(cudaStream_t s, const FbArg& fa, int grid, const AdamScalars& sc, const DevScalars* dyn,
                 uint64_t epoch, const BarrierArg& bar);

// K7 tcgen05 GEMM (gemm.cu): C[M,N] (+)= A[M,K]·B[K,N], bf16 operands K- or MN-major,
// fp32 accumulation; planned once (TMA descriptors encoded), launched many times.
struct GemmLaunch {
  CUtensorMap ma, mb, mc;
  alignas(8) unsigned char params[64];
  int ntiles = 0, grid = 1;
  double flops = 0;
};
GemmLaunch plan_gemm(const void* a, uint64_t lda, int a_mn, const void* b, uint64_t ldb, int b_mn, void* c,
                     uint64_t ldc, mics_dtype c_t, int M, int N, int K, int accumulate, int max_sms = 0);
void launch_gemm(cudaStream_t s, const GemmLaunch& g);

AdamScalars make_adam_scalars(double lr, double b1, double b2, double eps, double wd, int step, double grad_scale);

}  // namespace mics

// --------------------------------------------------------------------------
// the context (VirtualRankEngine's B200 counterpart)
struct mics_ctx {
  int n = 0, world = 1, wrank = 0, per = 0, device = 0, nsm = 148;
  // Single-process multi-GPU context (mics_init_devices): `subs` holds one member
  // context per GPU — member d behaves as process d of a `world`-GPU job, with its own
  // arena, streams and barrier slots, peers mapped by peer access instead of CUDA IPC.
  // Every C-ABI call on the group is run member by member (capi.cpp): each plans and
  // enqueues the work of its own ranks, and the device flag barriers synchronise them,
  // exactly as the separate processes of a torchrun job are synchronised.
  std::vector<mics_ctx*> subs;
  bool member = false;  // a member of a group (host-buffer staging allowed although world > 1)
  int blocks_per_sm = 4;
  // resident CTAs/SM per kernel: copy, adam, reduce by [input dtype][source class 2/4/8/9]
  int occ_copy = 2, occ_adam = 4, occ_reduce[4][4] = {};
  int occ_copy_indep = 1;  // CTAs/SM of barrier-free gathers chained with PDL
  int occ_hier = 2;        // CTAs/SM of the one-launch hierarchical all-gather (one resident wave)
  int occ_fbnd = 2;        // CTAs/SM of the fused layer-group boundary (one resident wave)
  int bar_strict = 0;      // BarrierArg::strict (MICS_BAR_STRICT)
  int par_ctas_per_sm = 0; // mics_set_parallelism: CTAs per SM cap (0 = occupancy)
  int par_max_ctas = 0;    // mics_set_parallelism: CTAs per launch cap (0 = none)
  int reduce_occ(mics_dtype t, uint32_t max_p) const {
    const int pc = mics::reduce_class(max_p);
    return occ_reduce[t][pc == 2 ? 0 : pc == 4 ? 1 : pc == 8 ? 2 : 3];
  }
  cudaStream_t stream = nullptr;
  // Barrier channels: each has its own flag slots, pairwise counters and CTA
  // tickets, so two streams can run barrier kernels concurrently (channel c is
  // only ever used from one stream, in the same order on every process).
  // 0: main stream; 1: side stream (the overlapped tail's Adam) or the compute step's
  // gather stream; 2: the tail's boundary reduce-scatter stream or the compute step's
  // copy-engine reduce-scatter barriers.  Each channel is driven by one stream per step.
  static constexpr int kChannels = 3;
  cudaStream_t side_stream = nullptr;  // channel 1: the overlapped tail's Adam
  char* base = nullptr;           // local arena (IPC-exportable)
  uint64_t cap = 0, used = 0;
  uint64_t top = 0;  // [top, cap): long-lived symmetric regions carved from the arena's end (hier_flags)
  char* peer_base[MICS_MAX_WORLD] = {};
  bool ipc_ready = false;
  mics::PeerTab* d_tab = nullptr;   // [kChannels]
  uint64_t* d_nbar = nullptr;       // [kChannels][MICS_MAX_WORLD]
  unsigned* d_tickets = nullptr;    // [kChannels][2]
  mics::HierCtl* d_hctl = nullptr;  // [kChannels] hierarchical all-gather epochs
  mics_buf hflags{};                // stage-1 tile flags of ad-hoc hierarchical all-gathers (grown on demand)
  // descriptor ring for ad-hoc calls
  char* ring = nullptr;
  uint64_t ring_cap = 0, ring_head = 0;
  bool traffic_on = true;
  std::map<std::pair<int, int>, uint64_t> traffic;
  uint64_t launches = 0;

  int process_of(int rank) const { return rank / per; }
  bool local(int rank) const { return process_of(rank) == wrank; }
  char* rank_ptr(mics_buf b, int rank) const {
    return peer_base[process_of(rank)] + b.offset + uint64_t(rank % per) * b.stride;
  }
  void record(int from, int to, uint64_t bytes) {
    if (!traffic_on) return;
    if (world > 1 && !local(to)) return;
    traffic[{from, to}] += bytes;
  }
  int grid_for(uint64_t tiles, int per_sm = 0) const {
    int k = per_sm ? per_sm : blocks_per_sm;
    if (par_ctas_per_sm > 0 && par_ctas_per_sm < k) k = par_ctas_per_sm;
    uint64_t g = uint64_t(nsm) * uint64_t(k);
    if (par_max_ctas > 0 && uint64_t(par_max_ctas) < g) g = uint64_t(par_max_ctas);
    if (tiles < g) g = tiles;
    return g ? int(g) : 1;
  }
  // device memory for descriptor tables of one ad-hoc launch
  void* ring_put(const void* host, uint64_t bytes);
  void* ring_reserve(uint64_t bytes);
  void ring_upload(void* dev, const void* host, uint64_t bytes);
  mics::BarrierArg barrier(uint64_t mask, int entry, int exit, int chan = 0, int publish = 1) const {
    mics::BarrierArg b;
    b.tab = d_tab + chan;
    b.nbar = d_nbar + chan * MICS_MAX_WORLD;
    b.tickets = d_tickets + 2 * chan;
    b.mask = ipc_ready ? mask : 0;
    b.entry = entry;
    b.exit = exit;
    b.dep_first = 1;
    b.strict = bar_strict;
    b.publish = publish;
    return b;
  }
  // processes hosting any of `ranks`, minus self (0 when self hosts none)
  uint64_t peer_mask(const int* ranks, int count) const;
  bool is_local_ptr(const void* p) const {
    const char* c = static_cast<const char*>(p);
    return !ipc_ready || (c >= base && c < base + cap);
  }
  uint64_t local_alloc(uint64_t bytes);  // world == 1 (or group member) scratch
};

namespace mics {
// the contexts that run a call: the members of a multi-device group, or the context itself
inline std::vector<mics_ctx*> members(mics_ctx* c) { return c->subs.empty() ? std::vector<mics_ctx*>{c} : c->subs; }
// the member hosting `rank` (the context itself when it is not a group)
inline mics_ctx* owner(mics_ctx* c, int rank) {
  return c->subs.empty() ? c : c->subs[size_t(c->process_of(rank))];
}
// collectives planners (collectives.cpp), shared with the sync/step drivers
struct CopyPlan {
  std::vector<CopySeg> segs;
  uint32_t tiles = 0;
  void add(const void* src, const std::vector<void*>& dsts, uint64_t bytes);
  // A stripe group: equal-size copies whose tiles are interleaved (tile t of the
  // group belongs to copy t mod k), so every source — local HBM and each NVLink
  // peer — is read concurrently instead of one after the other.
  void add_group(const std::vector<std::pair<const void*, std::vector<void*>>>& items, uint64_t bytes);
};
struct RedPlan {
  std::vector<RedJob> jobs;
  std::vector<std::vector<const void*>> srcs;  // per job
  uint32_t tiles = 0;
  uint32_t tile_elems = 0;
  uint32_t max_p = 1;
  explicit RedPlan(mics_dtype in_t) : tile_elems(reduce_tile_elems(in_t)) {}
  void add(const std::vector<const void*>& src, void* dst, uint64_t elems, uint64_t valid);
};
// One hierarchical all-gather (K3) over every partition group of an n-rank cluster:
// stage-1 then stage-3 segments of every local rank (HierSeg).
struct HierPlan {
  std::vector<HierSeg> segs;
  uint32_t tiles = 0;
  bool sys = false;  // a node peer of a local rank lives in another process
  uint64_t remote_bytes = 0, hbm_bytes = 0;
  // items: (src, dst, flags); equal sizes, tiles interleaved (stripe group)
  void add_group(int stage, const std::vector<std::tuple<const void*, void*, uint64_t*>>& items, uint64_t bytes,
                 int lag = 0);
};
// The ad-hoc hierarchical all-gathers' flag array (>= bytes per rank, zeroed), carved
// from the top of the arena so mark/release of the bump allocator never frees it.
mics_buf hier_flags(mics_ctx* ctx, uint64_t bytes_per_rank);
// Tiles per chunk of the flag array of one rank: q chunks x this many u64 flags.
inline uint64_t hier_flag_tiles(uint64_t chunk_bytes) { return ceil_div(chunk_bytes, kCopyTile); }
// src(r): rank r's input chunk; dst(r, pos): position `pos` of rank r's output; flags(r):
// rank r's flag array ([q][ftiles] u64, peer-mapped for remote ranks).
// stages: bit 0 = stage 1, bit 1 = stage 3; lag: see HierSeg::lag
HierPlan plan_hier(mics_ctx* ctx, int n, int p, int k, uint64_t chunk, int corrupt,
                   const std::function<const void*(int)>& src, const std::function<char*(int, uint64_t)>& dst,
                   const std::function<uint64_t*(int)>& flags, uint64_t ftiles, int stages = 3, int lag = 0);
// the segments of `b` after those of `a`, in one launch
HierPlan concat_hier(const HierPlan& a, const HierPlan& b);
struct AdamPlan {
  std::vector<AdamJob> jobs;
  std::vector<std::vector<const void*>> srcs;
  uint32_t tiles = 0;
  void add(const std::vector<const void*>& src, float* param, float* m, float* v, uint16_t* pbf16, float* gout,
           uint64_t elems, uint64_t sub);
  // the job just added also updates a second replica (param2, m2, v2, pbf16_2)
  void add_replica(float* param2, float* m2, float* v2, uint16_t* pbf16_2);
};

// A device-resident, replayable launch (built once, launched many times).
struct Launch {
  enum Kind { COPY, REDUCE, ADAM, BARRIER, TAIL, HIER, FBND } kind = COPY;
  int tail_r = 0, tail_p = 0;  // TAIL: replicas and group size (mode = 1 zero-accumulate)
  int hier_sys = 0, hier_chan = 0;  // HIER: system-scope flags; channel of its epoch counter
  uint64_t hier_peers = 0;          // HIER (merged): processes whose previous launch lag-1 tiles read
  int hier_merged = 0;              // HIER: merged launch (done counter instead of per-tile flags)
  uint32_t hier_n1 = 0;             // HIER (merged): stage-1 tiles, interleaved with the stage-3 tiles
  FbArg fb;                         // FBND: the launch's tables and shape
  uint64_t fb_epoch = 0;            // FBND: flag value (eager launches; graph replays read DevScalars)
  void* d_desc = nullptr;  // owned device table (cudaMalloc)
  uint64_t table_bytes = 0;
  uint32_t max_p = 1;
  int ndesc = 0;
  uint32_t ntiles = 0;
  int grid = 1;
  mics_dtype in_t = MICS_F32, acc_t = MICS_F32;
  double scale = 1.0;
  int mode = 0;
  AdamScalars adam{};
  const DevScalars* dyn = nullptr;  // ADAM/TAIL: per-step scalars in device memory (graph replay)
  BarrierArg bar{};
  // algorithmic bytes one launch moves on this GPU: pulled from peers over NVLink,
  // and local HBM reads + writes (the roofline numerators of bench.py)
  uint64_t remote_bytes = 0, hbm_bytes = 0;
  void release();
};
Launch make_copy_launch(mics_ctx* ctx, const CopyPlan& plan, const BarrierArg& bar, bool persistent);
// chan: barrier channel whose HierCtl epoch counter the launch advances
Launch make_hier_launch(mics_ctx* ctx, const HierPlan& plan, const BarrierArg& bar, int chan, bool persistent);
Launch make_reduce_launch(mics_ctx* ctx, const RedPlan& plan, mics_dtype in_t, mics_dtype acc_t, double scale, int mode,
                          const BarrierArg& bar, bool persistent);
Launch make_adam_launch(mics_ctx* ctx, const AdamPlan& plan, const AdamScalars& sc, const BarrierArg& bar,
                        bool persistent);
// dep_first: -1 = as planned, 0/1/2 = override BarrierArg::dep_first for this launch
void enqueue(mics_ctx* ctx, const Launch& l, int dep_first = -1, cudaStream_t stream = nullptr);

void check_group(const mics_ctx* ctx, const int* ranks, int p);
}  // namespace mics
