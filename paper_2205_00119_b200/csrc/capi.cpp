// The C-ABI edge (include/mics.h): exceptions never cross it.  Every entry point
// maps mics::Error to its status and keeps "<Errc>: detail" in a thread-local
// string, the way sdpsim::raise builds Error::what() (errors.hpp:32-34).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "internal.h"
#include "sync.h"

namespace mics {
// runtime.cpp
mics_ctx* create_ctx(const mics_init_args* a);
void destroy_ctx(mics_ctx* c);
void ipc_export(mics_ctx* c, void* handle);
void ipc_import(mics_ctx* c, const void* handles);
void barrier_all(mics_ctx* c);
// topology.cpp
void cluster_validate(const mics_cluster* c);
void build_group_layout(int n, int p, int* part, int* repl);
bool partition_shape_ok(int p, int k);
uint64_t model_state_bytes(uint64_t params, uint64_t bpp);
int min_feasible_partition(uint64_t states, const mics_cluster* c, bool node_granular, double headroom);
// collectives.cpp
void all_gather(mics_ctx*, const int*, int, const void* const*, uint64_t, void* const*);
void reduce_scatter(mics_ctx*, const int*, int, const void* const*, uint64_t, uint64_t, mics_dtype, mics_dtype, double,
                    int, void* const*);
void all_reduce(mics_ctx*, const int*, int, void* const*, uint64_t, mics_dtype);
void hier_all_gather(mics_ctx*, int, int, int, const void* const*, uint64_t, void* const*, int);
void batched_all_gather(mics_ctx*, const mics_ag_desc*, int);
void batched_reduce_scatter(mics_ctx*, const mics_rs_desc*, int, mics_dtype, mics_dtype, double, int);
void host_all_gather(mics_ctx*, const int*, int, const void* const*, uint64_t, void* const*);
void host_reduce_scatter(mics_ctx*, const int*, int, const void* const*, uint64_t, mics_dtype, void* const*);
void host_all_reduce(mics_ctx*, const int*, int, const void* const*, uint64_t, mics_dtype, void* const*);
void host_hier_all_gather(mics_ctx*, int, int, int, const void* const*, uint64_t, void* const*, int);
void host_batched_all_gather(mics_ctx*, int, const int*, const int*, const uint64_t*, const void* const*,
                             void* const*);
void host_batched_reduce_scatter(mics_ctx*, int, const int*, const int*, const uint64_t*, const void* const*,
                                 mics_dtype, void* const*);
Launch build_all_gather(mics_ctx*, const int*, int, const void* const*, uint64_t, void* const*, bool);
Launch build_reduce_scatter(mics_ctx*, const int*, int, const void* const*, uint64_t, uint64_t, mics_dtype,
                            mics_dtype, double, int, void* const*, bool);
// step.cpp
mics_step* step_create(mics_ctx* ctx, const mics_step_cfg* cfg);
void step_destroy(mics_step* st);
void step_run(mics_step* st, int iters);
void step_profile(mics_step* st, double* ms5);
void step_run_host(mics_step* st, const void* host_grads, int iters, void* host_result);
}  // namespace mics

struct mics_plan {
  std::vector<mics::Launch> launches;
};

namespace {
thread_local std::string g_last_error;

// build a persistent launch without logging traffic (a plan is not a transfer)
template <typename F>
mics_plan* make_plan(mics_ctx* ctx, F&& build) {
  const bool was = ctx->traffic_on;
  ctx->traffic_on = false;
  auto* p = new mics_plan();
  try {
    p->launches.push_back(build());
  } catch (...) {
    ctx->traffic_on = was;
    delete p;
    throw;
  }
  ctx->traffic_on = was;
  return p;
}

template <typename F>
mics_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return MICS_OK;
  } catch (const mics::Error& e) {
    g_last_error = e.what;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = std::string("ConfigError: ") + e.what();
    return MICS_CONFIG_ERROR;
  }
}

void need(const void* p, const char* what) {
  if (!p) mics::raise(MICS_OUT_OF_RANGE, std::string("null ") + what);
}
}  // namespace

extern "C" {

const char* mics_status_name(mics_status s) {
  switch (s) {
    case MICS_OK: return "Ok";
    case MICS_OUT_OF_RANGE: return "OutOfRange";
    case MICS_NON_DIVISIBLE: return "NonDivisible";
    case MICS_INFEASIBLE: return "Infeasible";
    case MICS_SIZE_MISMATCH: return "SizeMismatch";
    case MICS_TYPE_MISMATCH: return "TypeMismatch";
    case MICS_SHAPE_ERROR: return "ShapeError";
    case MICS_BOUNDARY_VIOLATION: return "BoundaryViolation";
    case MICS_EMPTY_PROFILE: return "EmptyProfile";
    case MICS_CONFIG_ERROR: return "ConfigError";
    case MICS_CUDA_ERROR: return "CudaError";
  }
  return "Unknown";
}

const char* mics_last_error(void) { return g_last_error.c_str(); }
int mics_abi_version(void) { return MICS_ABI_VERSION; }

// ---- topology
mics_status mics_build_group_layout(int n, int p, int* part, int* repl) {
  return guard([&] { mics::build_group_layout(n, p, part, repl); });
}
int mics_partition_shape_ok(int p, int k) { return mics::partition_shape_ok(p, k) ? 1 : 0; }
mics_status mics_model_state_bytes(uint64_t params, uint64_t bpp, uint64_t* out) {
  return guard([&] {
    need(out, "output");
    *out = mics::model_state_bytes(params, bpp);
  });
}
mics_status mics_cluster_validate(const mics_cluster* c) { return guard([&] { mics::cluster_validate(c); }); }
mics_status mics_min_feasible_partition(uint64_t states, const mics_cluster* c, int node_granular, double headroom,
                                        int* p_out) {
  return guard([&] {
    need(p_out, "output");
    *p_out = mics::min_feasible_partition(states, c, node_granular != 0, headroom);
  });
}

// ---- context
mics_status mics_init(const mics_init_args* args, mics_ctx** out) {
  return guard([&] {
    need(out, "output");
    *out = mics::create_ctx(args);
  });
}
mics_status mics_destroy(mics_ctx* ctx) { return guard([&] { mics::destroy_ctx(ctx); }); }
mics_status mics_ipc_export(mics_ctx* ctx, void* handle) {
  return guard([&] {
    need(ctx, "ctx");
    need(handle, "handle");
    mics::ipc_export(ctx, handle);
  });
}
mics_status mics_ipc_import(mics_ctx* ctx, const void* handles) {
  return guard([&] {
    need(ctx, "ctx");
    need(handles, "handles");
    mics::ipc_import(ctx, handles);
  });
}
mics_status mics_rank_process(mics_ctx* ctx, int rank, int* w) {
  return guard([&] {
    need(ctx, "ctx");
    need(w, "output");
    if (rank < 0 || rank >= ctx->n) mics::raise(MICS_OUT_OF_RANGE, "rank out of range");
    *w = ctx->process_of(rank);
  });
}
mics_status mics_local_ranks(mics_ctx* ctx, int* first, int* count) {
  return guard([&] {
    need(ctx, "ctx");
    if (first) *first = ctx->wrank * ctx->per;
    if (count) *count = ctx->per;
  });
}
mics_status mics_set_parallelism(mics_ctx* ctx, int ctas_per_sm, int max_ctas) {
  return guard([&] {
    need(ctx, "ctx");
    if (ctas_per_sm < 0 || max_ctas < 0) mics::raise(MICS_OUT_OF_RANGE, "parallelism must be >= 0");
    ctx->par_ctas_per_sm = ctas_per_sm;
    ctx->par_max_ctas = max_ctas;
  });
}
mics_status mics_alloc(mics_ctx* ctx, uint64_t bytes, mics_buf* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = mics::alloc_sym(ctx, bytes);
  });
}
mics_status mics_arena_mark(mics_ctx* ctx, uint64_t* mark) {
  return guard([&] {
    need(ctx, "ctx");
    need(mark, "output");
    *mark = ctx->used;
  });
}
mics_status mics_arena_release(mics_ctx* ctx, uint64_t mark) {
  return guard([&] {
    need(ctx, "ctx");
    if (mark > ctx->used) mics::raise(MICS_OUT_OF_RANGE, "mark beyond the arena head");
    MICS_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->used = mark < 4096 ? 4096 : mark;
  });
}
mics_status mics_arena_used(mics_ctx* ctx, uint64_t* used, uint64_t* capacity) {
  return guard([&] {
    need(ctx, "ctx");
    if (used) *used = ctx->used;
    if (capacity) *capacity = ctx->top;  // what the bump allocator may use
  });
}
mics_status mics_buf_ptr(mics_ctx* ctx, mics_buf buf, int rank, void** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    mics::check_buf_rank(ctx, buf, rank, 0, 0);
    if (!ctx->peer_base[ctx->process_of(rank)]) mics::raise(MICS_CONFIG_ERROR, "peer arena not imported");
    *out = ctx->rank_ptr(buf, rank);
  });
}
mics_status mics_memset(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, int value, uint64_t bytes) {
  return guard([&] {
    need(ctx, "ctx");
    mics::check_buf_rank(ctx, buf, rank, off, bytes);
    if (!ctx->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "memset of a rank hosted by another process");
    MICS_CUDA(cudaMemsetAsync(ctx->rank_ptr(buf, rank) + off, value, bytes, ctx->stream));
  });
}
mics_status mics_h2d(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, const void* host, uint64_t bytes) {
  return guard([&] {
    need(ctx, "ctx");
    mics::check_buf_rank(ctx, buf, rank, off, bytes);
    if (!ctx->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "h2d into a rank hosted by another process");
    if (bytes) {
      need(host, "host buffer");
      MICS_CUDA(cudaMemcpyAsync(ctx->rank_ptr(buf, rank) + off, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
  });
}
mics_status mics_d2h(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, void* host, uint64_t bytes) {
  return guard([&] {
    need(ctx, "ctx");
    mics::check_buf_rank(ctx, buf, rank, off, bytes);
    if (!ctx->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "d2h from a rank hosted by another process");
    if (bytes) {
      need(host, "host buffer");
      MICS_CUDA(cudaMemcpyAsync(host, ctx->rank_ptr(buf, rank) + off, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      MICS_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}
mics_status mics_stream(mics_ctx* ctx, void** s) {
  return guard([&] {
    need(ctx, "ctx");
    need(s, "output");
    *s = ctx->stream;
  });
}
mics_status mics_synchronize(mics_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    MICS_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}
mics_status mics_barrier(mics_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    mics::barrier_all(ctx);
  });
}
mics_status mics_launch_count(mics_ctx* ctx, uint64_t* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = ctx->launches;
  });
}
mics_status mics_num_sms(mics_ctx* ctx, int* sms) {
  return guard([&] {
    need(ctx, "ctx");
    need(sms, "output");
    *sms = ctx->nsm;
  });
}
mics_status mics_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    need(out, "output");
    MICS_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}
mics_status mics_host_free(void* p) {
  return guard([&] { MICS_CUDA(cudaFreeHost(p)); });
}

// ---- traffic
mics_status mics_traffic_enable(mics_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->traffic_on = on != 0;
  });
}
mics_status mics_traffic_clear(mics_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->traffic.clear();
  });
}
mics_status mics_traffic_size(mics_ctx* ctx, uint64_t* entries) {
  return guard([&] {
    need(ctx, "ctx");
    need(entries, "output");
    *entries = ctx->traffic.size();
  });
}
mics_status mics_traffic_get(mics_ctx* ctx, int64_t* t, uint64_t cap) {
  return guard([&] {
    need(ctx, "ctx");
    uint64_t i = 0;
    for (const auto& [key, bytes] : ctx->traffic) {
      if (i >= cap) break;
      t[3 * i + 0] = key.first;
      t[3 * i + 1] = key.second;
      t[3 * i + 2] = int64_t(bytes);
      ++i;
    }
  });
}

// ---- collectives
mics_status mics_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* d_shard, uint64_t chunk,
                            void* const* d_out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::all_gather(ctx, ranks, p, d_shard, chunk, d_out);
  });
}
mics_status mics_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* d_in, uint64_t in_elems,
                                uint64_t valid, mics_dtype in_t, mics_dtype acc_t, double scale, mics_rs_mode mode,
                                void* const* d_out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::reduce_scatter(ctx, ranks, p, d_in, in_elems, valid, in_t, acc_t, scale, int(mode), d_out);
  });
}
mics_status mics_all_reduce(mics_ctx* ctx, const int* ranks, int p, void* const* buf, uint64_t elems, mics_dtype dt) {
  return guard([&] {
    need(ctx, "ctx");
    mics::all_reduce(ctx, ranks, p, buf, elems, dt);
  });
}
mics_status mics_hier_all_gather(mics_ctx* ctx, int p, int k, const void* const* d_shard, uint64_t chunk,
                                 void* const* d_out, int corrupt) {
  return guard([&] {
    need(ctx, "ctx");
    mics::hier_all_gather(ctx, ctx->n, p, k, d_shard, chunk, d_out, corrupt);
  });
}
mics_status mics_batched_all_gather(mics_ctx* ctx, const mics_ag_desc* d, int count) {
  return guard([&] {
    need(ctx, "ctx");
    mics::batched_all_gather(ctx, d, count);
  });
}
mics_status mics_batched_reduce_scatter(mics_ctx* ctx, const mics_rs_desc* d, int count, mics_dtype in_t,
                                        mics_dtype acc_t, double scale, mics_rs_mode mode) {
  return guard([&] {
    need(ctx, "ctx");
    mics::batched_reduce_scatter(ctx, d, count, in_t, acc_t, scale, int(mode));
  });
}
mics_status mics_plan_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* d_shard, uint64_t chunk,
                                 void* const* d_out, mics_plan** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = make_plan(ctx, [&] { return mics::build_all_gather(ctx, ranks, p, d_shard, chunk, d_out, true); });
  });
}
mics_status mics_plan_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* d_in,
                                     uint64_t in_elems, uint64_t valid, mics_dtype in_t, mics_dtype acc_t,
                                     double scale, mics_rs_mode mode, void* const* d_out, mics_plan** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = make_plan(ctx, [&] {
      return mics::build_reduce_scatter(ctx, ranks, p, d_in, in_elems, valid, in_t, acc_t, scale, int(mode), d_out,
                                        true);
    });
  });
}
mics_status mics_plan_run(mics_ctx* ctx, mics_plan* plan, int iterations) {
  return guard([&] {
    need(ctx, "ctx");
    need(plan, "plan");
    for (int i = 0; i < iterations; ++i)
      for (const auto& l : plan->launches) mics::enqueue(ctx, l);
  });
}
mics_status mics_plan_destroy(mics_plan* plan) {
  return guard([&] {
    if (!plan) return;
    for (auto& l : plan->launches) l.release();
    delete plan;
  });
}
mics_status mics_host_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* shards, uint64_t chunk,
                                 void* const* out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::host_all_gather(ctx, ranks, p, shards, chunk, out);
  });
}
mics_status mics_host_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* bufs, uint64_t bytes,
                                     mics_dtype dt, void* const* out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::host_reduce_scatter(ctx, ranks, p, bufs, bytes, dt, out);
  });
}
mics_status mics_host_all_reduce(mics_ctx* ctx, const int* ranks, int p, const void* const* bufs, uint64_t bytes,
                                 mics_dtype dt, void* const* out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::host_all_reduce(ctx, ranks, p, bufs, bytes, dt, out);
  });
}
mics_status mics_host_hier_all_gather(mics_ctx* ctx, int n, int p, int k, const void* const* shards, uint64_t chunk,
                                      void* const* out, int corrupt) {
  return guard([&] {
    need(ctx, "ctx");
    mics::host_hier_all_gather(ctx, n, p, k, shards, chunk, out, corrupt);
  });
}
mics_status mics_host_batched_all_gather(mics_ctx* ctx, int count, const int* sizes, const int* ranks,
                                         const uint64_t* chunks, const void* const* shards, void* const* out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::host_batched_all_gather(ctx, count, sizes, ranks, chunks, shards, out);
  });
}
mics_status mics_host_batched_reduce_scatter(mics_ctx* ctx, int count, const int* sizes, const int* ranks,
                                             const uint64_t* bytes, const void* const* bufs, mics_dtype dt,
                                             void* const* out) {
  return guard([&] {
    need(ctx, "ctx");
    mics::host_batched_reduce_scatter(ctx, count, sizes, ranks, bytes, bufs, dt, out);
  });
}

// ---- sync schedule
mics_status mics_sync_create(mics_ctx* ctx, int p, int s, int nseg, const uint64_t* seg_len, mics_dtype acc_t,
                             uint32_t align, mics_sync** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = mics::sync_create(ctx, p, s, nseg, seg_len, acc_t, align);
  });
}
mics_status mics_sync_destroy(mics_sync* st) {
  return guard([&] { delete st; });
}
mics_status mics_sync_get_info(mics_sync* st, mics_sync_info* info) {
  return guard([&] {
    need(st, "sync");
    need(info, "output");
    info->n = st->n;
    info->p = st->p;
    info->s = st->s;
    info->nseg = st->nseg;
    info->micro_step = st->micro_step;
    info->acc_t = st->acc_t;
    info->shard_elems = st->shard_elems;
    info->grad_elems = st->grad_elems;
    info->boundary_sub = st->sub;
    info->shard = st->shard;
  });
}
mics_status mics_sync_seg(mics_sync* st, int seg, uint64_t* len, uint64_t* chunk, uint64_t* shard_off,
                          uint64_t* grad_off) {
  return guard([&] {
    need(st, "sync");
    if (seg < 0 || seg >= st->nseg) mics::raise(MICS_OUT_OF_RANGE, "segment out of range");
    if (len) *len = st->len[size_t(seg)];
    if (chunk) *chunk = st->chunk[size_t(seg)];
    if (shard_off) *shard_off = st->shard_off[size_t(seg)];
    if (grad_off) *grad_off = st->grad_off[size_t(seg)];
  });
}
mics_status mics_sync_micro_step(mics_ctx* ctx, mics_sync* st, mics_buf grads, uint64_t off, mics_dtype grad_t,
                                 double scale, mics_rs_mode mode) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    mics::micro_step(st, grads, off, grad_t, scale, int(mode));
  });
}
mics_status mics_sync_boundary(mics_ctx* ctx, mics_sync* st, const mics_adam* adam) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    mics::boundary(st, adam);
  });
}
mics_status mics_sync_alt_step(mics_ctx* ctx, mics_sync* st, mics_buf grads, uint64_t off, mics_dtype grad_t,
                               double scale) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    mics::alt_step(st, grads, off, grad_t, scale);
  });
}
mics_status mics_sync_alt_boundary(mics_ctx* ctx, mics_sync* st) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    mics::alt_boundary(st);
  });
}
mics_status mics_sync_events(mics_sync* st, int64_t* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    need(st, "sync");
    if (count) *count = st->events.size();
    for (uint64_t i = 0; i < st->events.size() && i < cap; ++i)
      for (int k = 0; k < 4; ++k) out[4 * i + uint64_t(k)] = st->events[i][size_t(k)];
  });
}
mics_status mics_sync_clear_events(mics_sync* st) {
  return guard([&] {
    need(st, "sync");
    st->events.clear();
  });
}

// ---- generator
mics_status mics_generate(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, mics_dtype dt, uint64_t seed, int step,
                          int layer, uint64_t start, uint64_t count) {
  return guard([&] {
    need(ctx, "ctx");
    if (dt != MICS_F32 && dt != MICS_BF16) mics::raise(MICS_TYPE_MISMATCH, "generator emits f32 or bf16");
    mics::check_buf_rank(ctx, buf, rank, off, count * mics::dtype_size(dt));
    if (!ctx->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "generate into a rank hosted by another process");
    mics::launch_generate(ctx->stream, ctx->rank_ptr(buf, rank) + off, dt, seed, rank, step, layer, start, count,
                          ctx->nsm * 8);
    ctx->launches++;
  });
}

// ---- step driver
mics_status mics_step_create(mics_ctx* ctx, const mics_step_cfg* cfg, mics_step** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = mics::step_create(ctx, cfg);
  });
}
mics_status mics_step_destroy(mics_step* st) { return guard([&] { mics::step_destroy(st); }); }
mics_status mics_step_run(mics_ctx* ctx, mics_step* st, int iters) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    mics::step_run(st, iters);
  });
}
mics_status mics_step_stats_get(mics_step* st, mics_step_stats* out) {
  return guard([&] {
    need(st, "step");
    need(out, "output");
    *out = st->stats;
  });
}
mics_status mics_step_sync(mics_step* st, mics_sync** out) {
  return guard([&] {
    need(st, "step");
    need(out, "output");
    *out = st->sync;
  });
}
mics_status mics_step_buffers(mics_step* st, mics_buf* pb, mics_buf* master, mics_buf* m, mics_buf* v, mics_buf* g,
                              mics_buf* grads) {
  return guard([&] {
    need(st, "step");
    if (pb) *pb = st->pbf16;
    if (master) *master = st->master;
    if (m) *m = st->m;
    if (v) *v = st->v;
    if (g) *g = st->gathered;
    if (grads) *grads = st->grads;
  });
}
mics_status mics_step_profile(mics_ctx* ctx, mics_step* st, double* ag, double* rs, double* bnd, double* gen) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    double ms[5];
    mics::step_profile(st, ms);
    if (ag) *ag = ms[0];
    if (rs) *rs = ms[1];
    if (bnd) *bnd = ms[2];
    if (gen) *gen = ms[3];
  });
}
mics_status mics_step_profile_ex(mics_ctx* ctx, mics_step* st, double* ms5) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    need(ms5, "ms5");
    mics::step_profile(st, ms5);
  });
}
mics_status mics_step_run_host(mics_ctx* ctx, mics_step* st, const void* host_grads, int iters, void* host_result) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    need(host_grads, "host gradients");
    mics::step_run_host(st, host_grads, iters, host_result);
  });
}

}  // extern "C"

mics_status mics_gemm_bf16(mics_ctx* ctx, const void* a, uint64_t lda, int a_mn, const void* b, uint64_t ldb, int b_mn,
                           void* c, uint64_t ldc, mics_dtype c_t, int m, int n, int k, int accumulate) {
  return guard([&] {
    need(ctx, "ctx");
    if (!a || !b || !c) mics::raise(MICS_OUT_OF_RANGE, "gemm: null operand");
    const mics::GemmLaunch g = mics::plan_gemm(a, lda, a_mn, b, ldb, b_mn, c, ldc, c_t, m, n, k, accumulate);
    mics::launch_gemm(ctx->stream, g);
    ctx->launches++;
  });
}
