/* mics.h — C-ABI of the B200-native MiCS communication hot path (libmics.so).
 *
 * Drop-in boundary for the reference's hot path (sdpsim, /root/reference/proj):
 * every entry point names the reference interface it replaces (file:line).  No
 * torch types, no exceptions across the boundary: every call returns a
 * mics_status and leaves "<Errc>: detail" in mics_last_error() (thread-local),
 * mirroring sdpsim::raise (errors.hpp:32-34).
 *
 * Process model: one process per GPU (world processes); n virtual ranks are laid
 * out node-major, n/world contiguous ranks per GPU (rank r lives on process
 * r / (n/world)), exactly the reference's rank numbering (topology.hpp:24-25).
 * Memory is a symmetric arena per process; peers map each other's arena through
 * CUDA IPC (mics_ipc_export / mics_ipc_import) and pull over NVLink/NVSwitch.
 * Collectives are SPMD: every process calls the same sequence; a process only
 * produces the outputs of ranks it hosts.  All work is enqueued on the
 * context's stream; mics_synchronize() waits for it.
 */
#ifndef MICS_H
#define MICS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MICS_ABI_VERSION 3
#define MICS_IPC_HANDLE_BYTES 64
#define MICS_MAX_WORLD 64
#define MICS_MAX_GROUP 1024

/* Errc order of errors.hpp:8-18, then the GPU-side additions. */
typedef enum {
  MICS_OK = 0,
  MICS_OUT_OF_RANGE = 1,
  MICS_NON_DIVISIBLE = 2,
  MICS_INFEASIBLE = 3,
  MICS_SIZE_MISMATCH = 4,
  MICS_TYPE_MISMATCH = 5,
  MICS_SHAPE_ERROR = 6,
  MICS_BOUNDARY_VIOLATION = 7,
  MICS_EMPTY_PROFILE = 8,
  MICS_CONFIG_ERROR = 9,
  MICS_CUDA_ERROR = 10
} mics_status;

/* DType (collectives.hpp:17) + bf16 (gradient/parameter storage; input only for reductions). */
typedef enum { MICS_I64 = 0, MICS_F32 = 1, MICS_F64 = 2, MICS_BF16 = 3 } mics_dtype;

typedef struct mics_ctx mics_ctx;
typedef struct mics_sync mics_sync;
typedef struct mics_step mics_step;

/* A symmetric allocation: rank r's region starts at
 * arena_base[process(r)] + offset + (r mod ranks_per_process) * stride. */
typedef struct {
  uint64_t offset;
  uint64_t stride;
} mics_buf;

/* ClusterSpec (topology.hpp:13-28). */
typedef struct {
  int num_nodes;
  int devices_per_node;
  double intra_node_bandwidth;
  double inter_node_bandwidth_per_node;
  double alpha_intra;
  double alpha_inter;
  uint64_t device_memory;
  double device_peak_flops;
} mics_cluster;

/* ---------------------------------------------------------------- errors */
const char* mics_status_name(mics_status s);       /* errc_name, errors.hpp:36-49 */
const char* mics_last_error(void);                 /* Error::what() of the last failure */
int mics_abi_version(void);

/* ---------------------------------------------------------------- topology (host only, no GPU) */
/* build_group_layout (topology.cpp:21-43): partition_groups[g*p+i] = g*p+i,
 * replication_groups[j*(n/p)+m] = j+m*p.  Both arrays hold n ints. */
mics_status mics_build_group_layout(int n, int p, int* partition_groups, int* replication_groups);
int mics_partition_shape_ok(int p, int k);                                         /* topology.cpp:45-49 */
mics_status mics_model_state_bytes(uint64_t num_params, uint64_t bytes_per_param,  /* topology.cpp:51-56 */
                                   uint64_t* out);
mics_status mics_cluster_validate(const mics_cluster* c);                          /* topology.cpp:7-19 */
mics_status mics_min_feasible_partition(uint64_t state_bytes, const mics_cluster* c, /* topology.cpp:58-84 */
                                        int node_granular, double headroom, int* p_out);

/* ---------------------------------------------------------------- context (VirtualRankEngine, collectives.hpp:42-62) */
typedef struct {
  int n_ranks;          /* virtual ranks in the job (n) */
  int world;            /* processes == GPUs taking part (1 = everything on this GPU) */
  int world_rank;       /* this process */
  int device;           /* CUDA ordinal of this process's GPU */
  uint64_t arena_bytes; /* symmetric arena per process (0 = 1 GiB) */
} mics_init_args;

mics_status mics_init(const mics_init_args* args, mics_ctx** out);
/* One process driving several GPUs (the reference's single in-process engine,
 * collectives.hpp:42-62, over NVLink): virtual ranks node-major over devices[0..ndev)
 * (rank r on devices[r / (n_ranks / ndev)]), peer access between every pair, one stream
 * per device, the same device flag barriers as a multi-process job.  args->world must
 * be 1.  Every other call takes the returned context like a single-GPU one; the
 * host-buffer API and the sync / step drivers then span the GPUs. */
mics_status mics_init_devices(const mics_init_args* args, const int* devices, int ndev, mics_ctx** out);
mics_status mics_device_count(mics_ctx* ctx, int* ndev); /* GPUs of the context (1 unless mics_init_devices) */
mics_status mics_device_stream(mics_ctx* ctx, int d, void** cuda_stream); /* member d's stream (timing) */
mics_status mics_destroy(mics_ctx* ctx);
/* CUDA IPC handle of this process's arena; gather all `world` handles (in world
 * order) with any out-of-band channel (torch.distributed) and import them. */
mics_status mics_ipc_export(mics_ctx* ctx, void* handle /* MICS_IPC_HANDLE_BYTES */);
mics_status mics_ipc_import(mics_ctx* ctx, const void* handles /* world * MICS_IPC_HANDLE_BYTES */);
mics_status mics_rank_process(mics_ctx* ctx, int rank, int* world_rank);
mics_status mics_local_ranks(mics_ctx* ctx, int* first, int* count);
/* The engine's worker count — VirtualRankEngine(num_threads) (collectives.hpp:42-47)
 * on the GPU: every collective planned from now on runs at most `ctas_per_sm` CTAs per
 * SM (0 = one resident wave at the kernel's occupancy) and at most `max_ctas` CTAs per
 * launch (0 = no cap).  Like the reference's thread count it changes only how the work
 * is spread: results and the traffic log are bit-identical for every setting
 * (collectives.hpp:38-41; tests/test_gpu_determinism.py). */
mics_status mics_set_parallelism(mics_ctx* ctx, int ctas_per_sm, int max_ctas);

/* Symmetric allocation: every process must make the same sequence of calls. */
mics_status mics_alloc(mics_ctx* ctx, uint64_t bytes_per_rank, mics_buf* out);
mics_status mics_arena_mark(mics_ctx* ctx, uint64_t* mark);
mics_status mics_arena_release(mics_ctx* ctx, uint64_t mark);
mics_status mics_arena_used(mics_ctx* ctx, uint64_t* used, uint64_t* capacity);
mics_status mics_buf_ptr(mics_ctx* ctx, mics_buf buf, int rank, void** out); /* local or peer-mapped */
mics_status mics_memset(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, int value, uint64_t bytes);
mics_status mics_h2d(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, const void* host, uint64_t bytes);
mics_status mics_d2h(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, void* host, uint64_t bytes);
mics_status mics_stream(mics_ctx* ctx, void** cuda_stream);
mics_status mics_synchronize(mics_ctx* ctx);
/* device-side flag barrier among all `world` processes (no host round trip) */
mics_status mics_barrier(mics_ctx* ctx);
mics_status mics_launch_count(mics_ctx* ctx, uint64_t* launches); /* kernels this ctx launched */
mics_status mics_num_sms(mics_ctx* ctx, int* sms);
mics_status mics_host_alloc(uint64_t bytes, void** out); /* pinned host memory (e2e inputs) */
mics_status mics_host_free(void* ptr);

/* traffic log (VirtualRankEngine::record_traffic / traffic, collectives.cpp:46-67).
 * Recorded analytically per message in the reference's own accounting; in a
 * multi-process job each process records the messages its ranks receive. */
mics_status mics_traffic_enable(mics_ctx* ctx, int on);
mics_status mics_traffic_clear(mics_ctx* ctx);
mics_status mics_traffic_size(mics_ctx* ctx, uint64_t* entries);
mics_status mics_traffic_get(mics_ctx* ctx, int64_t* triples /* (from,to,bytes) */, uint64_t cap);

/* ---------------------------------------------------------------- collectives on device memory
 * Arrays are indexed by group position (CollectiveGroup, collectives.hpp:30-36);
 * `ranks` are global virtual ranks.  Input pointers must be valid for every
 * position (peer pointers from mics_buf_ptr); output entries are used only for
 * ranks this process hosts.  The call enqueues one or two kernels; inputs may be
 * reused/overwritten once the call's work has completed on the stream (every
 * process in the group has finished reading them: exit barrier). */

/* all_gather (collectives.cpp:103-134): d_out[j] = d_shard[0] || ... || d_shard[p-1] */
mics_status mics_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* d_shard,
                            uint64_t chunk_bytes, void* const* d_out);

typedef enum {
  MICS_RS_STORE = 0,     /* out  = scale * fold           (reduce_scatter semantics) */
  MICS_RS_ACCUMULATE = 1,/* out  = out + scale * fold     (two_hop_micro_step :137-141) */
  MICS_RS_ZERO_ACCUM = 2 /* out  = 0 + scale * fold       (ACCUMULATE onto a zeroed shard, no memset) */
} mics_rs_mode;

/* reduce_scatter (collectives.cpp:136-183) fused with cast + scale + shard accumulate:
 * position j gets fold_{i=0..p-1}(cast(d_in[i][j*chunk + e])) in ascending position
 * order, starting from position 0's value (bit-exact with the reference).
 * in_elems = p*chunk per rank; elements at index >= valid_elems read as 0
 * (padded_grad, sync_schedule.hpp:105-111).  scale is applied once to the fold
 * (skipped when 1.0).  acc_t = in_t, or F32 for BF16 input. */
mics_status mics_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* d_in,
                                uint64_t in_elems, uint64_t valid_elems, mics_dtype in_t, mics_dtype acc_t,
                                double scale, mics_rs_mode mode, void* const* d_out);

/* all_reduce = reduce_scatter then all_gather (collectives.cpp:185-190), in place. elems % p == 0. */
mics_status mics_all_reduce(mics_ctx* ctx, const int* ranks, int p, void* const* d_buf, uint64_t elems,
                            mics_dtype dtype);

/* hierarchical_all_gather (collectives.cpp:192-291) over every partition group of
 * build_group_layout(n, p) with k ranks per (virtual) node; arrays have n entries
 * indexed by global rank.  Stage 2 is folded into the stage-1 store addressing;
 * corrupt_stage2 reproduces the reference's wrong-layout hook (:243-257). */
mics_status mics_hier_all_gather(mics_ctx* ctx, int p, int k, const void* const* d_shard, uint64_t chunk_bytes,
                                 void* const* d_out, int corrupt_stage2);

/* coalesced collectives (collectives.cpp:293-321; PAPER §4): one launch per call. */
typedef struct {
  const int* ranks;
  int p;
  const void* const* d_shard;
  uint64_t chunk_bytes;
  void* const* d_out;
} mics_ag_desc;
typedef struct {
  const int* ranks;
  int p;
  const void* const* d_in;
  uint64_t in_elems;
  uint64_t valid_elems;
  void* const* d_out;
} mics_rs_desc;
mics_status mics_batched_all_gather(mics_ctx* ctx, const mics_ag_desc* descs, int count);
mics_status mics_batched_reduce_scatter(mics_ctx* ctx, const mics_rs_desc* descs, int count, mics_dtype in_t,
                                        mics_dtype acc_t, double scale, mics_rs_mode mode);

/* Persistent (replayable) collectives: the descriptor table is built and uploaded
 * once; mics_plan_run enqueues the same kernel `iterations` times (hot loops, the
 * step driver, CUDA-graph capture).  Same semantics and barriers as the one-shot
 * calls; traffic is not logged per run. */
typedef struct mics_plan mics_plan;
mics_status mics_plan_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* d_shard,
                                 uint64_t chunk_bytes, void* const* d_out, mics_plan** out);
mics_status mics_plan_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* d_in,
                                     uint64_t in_elems, uint64_t valid_elems, mics_dtype in_t, mics_dtype acc_t,
                                     double scale, mics_rs_mode mode, void* const* d_out, mics_plan** out);
mics_status mics_plan_run(mics_ctx* ctx, mics_plan* plan, int iterations);
mics_status mics_plan_destroy(mics_plan* plan);

/* ---------------------------------------------------------------- host-buffer drop-ins
 * Same signatures as the reference's by-value API (collectives.hpp:64-112) over
 * host memory: H2D, kernel, D2H.  Single-process contexts (world == 1) only. */
mics_status mics_host_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* shards,
                                 uint64_t chunk_bytes, void* const* out);
mics_status mics_host_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* bufs,
                                     uint64_t bytes, mics_dtype dtype, void* const* out);
mics_status mics_host_all_reduce(mics_ctx* ctx, const int* ranks, int p, const void* const* bufs, uint64_t bytes,
                                 mics_dtype dtype, void* const* out);
mics_status mics_host_hier_all_gather(mics_ctx* ctx, int n, int p, int k, const void* const* shards,
                                      uint64_t chunk_bytes, void* const* out, int corrupt_stage2);
mics_status mics_host_batched_all_gather(mics_ctx* ctx, int count, const int* sizes, const int* ranks,
                                         const uint64_t* chunk_bytes, const void* const* shards, void* const* out);
mics_status mics_host_batched_reduce_scatter(mics_ctx* ctx, int count, const int* sizes, const int* ranks,
                                             const uint64_t* bytes, const void* const* bufs, mics_dtype dtype,
                                             void* const* out);

/* ---------------------------------------------------------------- 2-hop gradient sync (sync_schedule.hpp)
 * A mics_sync holds SyncState (sync_schedule.hpp:45-51) for every rank of the job:
 * the owned shard on the device (symmetric), micro_step and s.  Gradients are
 * `nseg` flat segments (nseg = 1 is the reference's single vector; the step driver
 * uses one per layer); segment i is sharded into p chunks of
 * chunk_i = ceil(len_i/p) rounded up to align_elems (1 = the reference's
 * owned_chunk_elems, :53-56).  The shard of a rank is the concatenation of its
 * chunks.  The gradient input of a rank is the concatenation of segments, each
 * laid out padded to p*chunk_i elements (padding is never read). */
typedef struct {
  int n, p, s, nseg;
  int micro_step;
  mics_dtype acc_t;
  uint64_t shard_elems;      /* sum of chunk_i */
  uint64_t grad_elems;       /* sum of p*chunk_i: gradient input elements per rank */
  uint64_t boundary_sub;     /* replication-group slice size used at the boundary */
  mics_buf shard;            /* accumulated owned shard, shard_elems (padded to r*boundary_sub) */
} mics_sync_info;

typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
  int step;                  /* 1-based Adam step (bias correction) */
  double grad_scale;         /* applied to the reduced gradient (e.g. 1/(n*s)) */
  mics_buf param;            /* fp32 master shard, shard_elems */
  mics_buf exp_avg;          /* fp32 */
  mics_buf exp_avg_sq;       /* fp32 */
  mics_buf param_bf16;       /* optional bf16 copy for the next all-gather (stride 0 = none) */
  int write_grad;            /* also leave the reduced gradient in the shard (reference AR semantics) */
} mics_adam;

mics_status mics_sync_create(mics_ctx* ctx, int p, int s, int nseg, const uint64_t* seg_len, mics_dtype acc_t,
                             uint32_t align_elems, mics_sync** out);
mics_status mics_sync_destroy(mics_sync* st);
mics_status mics_sync_get_info(mics_sync* st, mics_sync_info* info);
mics_status mics_sync_seg(mics_sync* st, int seg, uint64_t* len, uint64_t* chunk, uint64_t* shard_off,
                          uint64_t* grad_off);
/* two_hop_micro_step (:118-147): RS inside every partition group, shard (+)= result.
 * first micro-step of a window may use ZERO_ACCUM (state left from the previous
 * window is discarded) or ACCUMULATE (the reference keeps it). */
mics_status mics_sync_micro_step(mics_ctx* ctx, mics_sync* st, mics_buf grads, uint64_t grads_off,
                                 mics_dtype grad_t, double scale, mics_rs_mode mode);
/* two_hop_boundary (:153-185): AR inside every replication group; with adam != NULL
 * the AR's all-gather phase is fused with the sharded Adam update. */
mics_status mics_sync_boundary(mics_ctx* ctx, mics_sync* st, const mics_adam* adam);
/* alternative_schedule_step / alternative_boundary (:189-232): AR over all n ranks. */
mics_status mics_sync_alt_step(mics_ctx* ctx, mics_sync* st, mics_buf grads, uint64_t grads_off,
                               mics_dtype grad_t, double scale);
mics_status mics_sync_alt_boundary(mics_ctx* ctx, mics_sync* st);
/* SyncEvent log (:27-32): 4 int64 per event (step, phase, group, bytes). */
mics_status mics_sync_events(mics_sync* st, int64_t* out, uint64_t cap, uint64_t* count);
mics_status mics_sync_clear_events(mics_sync* st);

/* ---------------------------------------------------------------- synthetic gradients (K6)
 * x = splitmix64(seed ^ rank<<40 ^ step<<32 ^ layer<<24 ^ idx) -> f32 in [-1,1) (24 bits) or an
 * exactly-representable bf16 (8 bits); idx runs from `start`.  dtype F32 or BF16. */
/* K7: dense bf16 GEMM on the tcgen05 tensor cores (TMA + TMEM), the layer compute of
 * the step with compute (the reference has no GEMM: unpinned, checked
 * against an fp32 matmul).  C[m,n] (+)= sum_k A(m,k) B(k,n) on the ctx stream, device
 * pointers, row-major storage:
 *   A(m,k) = a[m*lda + k] (a_mn = 0, K-major) or a[k*lda + m] (a_mn = 1, M-major)
 *   B(k,n) = b[n*ldb + k] (b_mn = 0, K-major) or b[k*ldb + n] (b_mn = 1, N-major)
 *   C(m,n) = c[m*ldc + n], f32 or bf16 (RNE); accumulate = 1 adds into an f32 C.
 * a, b 16-byte aligned, lda/ldb multiples of 8. */
mics_status mics_gemm_bf16(mics_ctx* ctx, const void* a, uint64_t lda, int a_mn, const void* b, uint64_t ldb, int b_mn,
                           void* c, uint64_t ldc, mics_dtype c_t, int m, int n, int k, int accumulate);

mics_status mics_generate(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, mics_dtype dtype, uint64_t seed,
                          int step, int layer, uint64_t start, uint64_t count);

/* ---------------------------------------------------------------- MiCS step driver
 * One global step (simulator.cpp:265-280 order, executed for real):
 *   for t < s: per-layer parameter all-gather (fwd, layers 0..L-1),
 *              per-layer parameter all-gather (bwd, L-1..0),
 *              coalesced gradient reduce-scatter of all layers (2-hop hop 1);
 *   boundary:  replication-group all-reduce fused with sharded fp32 Adam (hop 2).
 * Parameters are bf16 shards (+ fp32 master, m, v), gathered into rotating
 * per-layer slots (3, or 2 with compute); gradients are pre-generated (resident) or produced per micro-step by
 * the K6 generator (models backward's gradient write). */
typedef struct {
  int p, s, nlayers;
  const uint64_t* layer_params;  /* parameters per layer */
  mics_dtype grad_t;             /* F32 or BF16 */
  int hier_k;                    /* 0 = flat all-gather, else ranks per virtual node */
  int resident_grads;            /* 1: s gradient sets generated once, before timing */
  int alternative;               /* 1: DeepSpeed-default global all-reduce every micro-step */
  uint64_t seed;
  double lr, beta1, beta2, eps, weight_decay;
  /* Step with compute (SURVEY 8f items 2+3; the reference has none).  Each layer l is a
   * linear map W_l = its gathered bf16 parameters viewed as [E_l / hidden, hidden]; every
   * layer reads the micro-step's input X [tokens, hidden] (bf16) and the loss is
   * 1/2 sum_l ||X W_l^T||^2, so per rank and micro-step: forward Y_l = X W_l^T, backward
   * dX += Y_l W_l and dW_l = Y_l^T X (tcgen05 GEMMs, K7), written as the layer's gradient
   * that the micro-step reduce-scatter consumes.  The gather of layer l+1 runs on its own
   * stream, overlapping layer l's GEMMs (prefetch depth 1, simulator.cpp:231-259); the
   * reduce-scatter of micro-step t overlaps micro-step t+1's compute. */
  int compute;                   /* 1: layer GEMMs in the step (gradients come from them) */
  int recompute;                 /* 1: recompute Y_l in the backward pass instead of storing it */
  uint64_t tokens;               /* rows of X per rank and micro-step (micro_batch * seq_len) */
  uint64_t hidden;               /* columns of X; every E_l must be a multiple */
} mics_step_cfg;

typedef struct {
  uint64_t ag_bytes_in;      /* NVLink/peer ingress per rank per step: parameter all-gathers */
  uint64_t rs_bytes_in;      /* per rank per step: micro-step reduce-scatters */
  uint64_t ar_bytes_in;      /* per rank per step: boundary all-reduce */
  uint64_t adam_hbm_bytes;   /* per rank per step: Adam state traffic */
  uint64_t gen_bytes;        /* per rank per step: gradient generation writes */
  uint64_t launches;         /* kernels per step (this process) */
  uint64_t shard_elems;
  uint64_t gathered_max_bytes;
  uint64_t grad_elems;
  int adam_step;
  /* this process, per step, summed from the planned descriptor tables: bytes pulled
   * from peers over NVLink and local HBM bytes (reads + writes), and launches, per phase */
  uint64_t ag_remote_bytes, ag_hbm_bytes, ag_launches;
  uint64_t rs_remote_bytes, rs_hbm_bytes, rs_launches;
  uint64_t bnd_remote_bytes, bnd_hbm_bytes, bnd_launches;
  /* step with compute: tensor-core FLOPs and GEMM launches per step (this process) */
  double compute_flops;
  uint64_t gemm_launches;
  uint64_t gather_slots;       /* layer l's gathered parameters live in slot l % gather_slots */
  uint64_t gather_slot_bytes;  /* bytes of one slot of the `gathered` buffer (per rank) */
} mics_step_stats;

mics_status mics_step_create(mics_ctx* ctx, const mics_step_cfg* cfg, mics_step** out);
mics_status mics_step_destroy(mics_step* st);
mics_status mics_step_run(mics_ctx* ctx, mics_step* st, int iterations); /* enqueue only */
mics_status mics_step_stats_get(mics_step* st, mics_step_stats* out);
mics_status mics_step_sync(mics_step* st, mics_sync** out);
mics_status mics_step_buffers(mics_step* st, mics_buf* param_bf16, mics_buf* master, mics_buf* exp_avg,
                              mics_buf* exp_avg_sq, mics_buf* gathered, mics_buf* grads);
/* per-phase kernel timing (CUDA events on the ctx stream) for the next run: ms per phase */
mics_status mics_step_profile(mics_ctx* ctx, mics_step* st, double* ag_ms, double* rs_ms, double* boundary_ms,
                              double* gen_ms);
/* per-phase device times of one serialised step: ms[0] all-gather, [1] reduce-scatter,
 * [2] boundary, [3] gradient generation, [4] layer GEMMs (step with compute) */
mics_status mics_step_profile_ex(mics_ctx* ctx, mics_step* st, double* ms5);
/* e2e variant: the step's inputs come from pinned HOST memory every micro-step (H2D in
 * the step): the gradients (grad_elems, reused per rank and micro-step), or with compute
 * the input X (tokens x hidden bf16) */
mics_status mics_step_run_host(mics_ctx* ctx, mics_step* st, const void* host_grads /* grad_elems, reused per rank/micro-step */,
                               int iterations, void* host_result /* per local rank: shard fp32, or NULL */);

#ifdef __cplusplus
}
#endif
#endif /* MICS_H */
