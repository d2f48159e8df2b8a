// The C-ABI edge (include/mics.h): exceptions never cross it.  Every entry point
// maps mics::Error to its status and keeps "<Errc>: detail" in a thread-local
// string, the way sdpsim::raise builds Error::what() (errors.hpp:32-34).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>

#include "internal.h"
#include "sync.h"

namespace mics {
// runtime.cpp
mics_ctx* create_ctx(const mics_init_args* a);
mics_ctx* create_group(const mics_init_args* a, const int* devices, int ndev);
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
mics_step* step_create(mics_ctx* ctx, const mics_step_cfg* cfg, bool settle = true);
ProfileRec* step_profile_begin(mics_step* st);
void step_profile_end(mics_step* st, ProfileRec* rec, double* ms);
void step_destroy(mics_step* st);
void step_run(mics_step* st, int iters);
void step_profile(mics_step* st, double* ms5);
void step_run_host(mics_step* st, const void* host_grads, int iters, void* host_result);
}  // namespace mics

struct mics_plan {
  std::vector<std::pair<mics_ctx*, mics::Launch>> launches;  // (member context, launch)
};

namespace {
thread_local std::string g_last_error;

// Run f(member) on every member context of `ctx` (itself when it is not a
// multi-device group), with that member's GPU current.
template <typename F>
void each(mics_ctx* ctx, F&& f) {
  for (mics_ctx* m : mics::members(ctx)) {
    MICS_CUDA(cudaSetDevice(m->device));
    f(m);
  }
}
// the member hosting `rank`, its GPU current
mics_ctx* at_rank(mics_ctx* ctx, int rank) {
  if (rank < 0 || rank >= ctx->n) mics::raise(MICS_OUT_OF_RANGE, "rank " + std::to_string(rank) + " out of range");
  mics_ctx* m = mics::owner(ctx, rank);
  MICS_CUDA(cudaSetDevice(m->device));
  return m;
}

// build persistent launches without logging traffic (a plan is not a transfer)
template <typename F>
mics_plan* make_plan(mics_ctx* ctx, F&& build) {
  auto* p = new mics_plan();
  try {
    each(ctx, [&](mics_ctx* m) {
      const bool was = m->traffic_on;
      m->traffic_on = false;
      try {
        p->launches.emplace_back(m, build(m));
      } catch (...) {
        m->traffic_on = was;
        throw;
      }
      m->traffic_on = was;
    });
  } catch (...) {
    for (auto& [m, l] : p->launches) l.release();
    delete p;
    throw;
  }
  return p;
}

// Every entry point: exceptions become a status, and the caller's current CUDA device
// is restored (a multi-device context switches devices member by member).
template <typename F>
mics_status guard(F&& f) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  struct Restore {
    int d;
    ~Restore() {
      if (d >= 0) cudaSetDevice(d);
    }
  } restore{dev};
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
mics_status mics_init_devices(const mics_init_args* args, const int* devices, int ndev, mics_ctx** out) {
  return guard([&] {
    need(out, "output");
    *out = mics::create_group(args, devices, ndev);
  });
}
mics_status mics_device_stream(mics_ctx* ctx, int d, void** s) {
  return guard([&] {
    need(ctx, "ctx");
    need(s, "output");
    const auto m = mics::members(ctx);
    if (d < 0 || d >= int(m.size())) mics::raise(MICS_OUT_OF_RANGE, "device index out of range");
    *s = m[size_t(d)]->stream;
  });
}
mics_status mics_device_count(mics_ctx* ctx, int* ndev) {
  return guard([&] {
    need(ctx, "ctx");
    need(ndev, "output");
    *ndev = ctx->subs.empty() ? 1 : int(ctx->subs.size());
  });
}
mics_status mics_destroy(mics_ctx* ctx) { return guard([&] { mics::destroy_ctx(ctx); }); }
mics_status mics_ipc_export(mics_ctx* ctx, void* handle) {
  return guard([&] {
    need(ctx, "ctx");
    need(handle, "handle");
    if (!ctx->subs.empty()) mics::raise(MICS_CONFIG_ERROR, "a multi-device context is one process: no IPC");
    mics::ipc_export(ctx, handle);
  });
}
mics_status mics_ipc_import(mics_ctx* ctx, const void* handles) {
  return guard([&] {
    need(ctx, "ctx");
    need(handles, "handles");
    if (!ctx->subs.empty()) mics::raise(MICS_CONFIG_ERROR, "a multi-device context is one process: no IPC");
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
    const bool group = !ctx->subs.empty();  // one process hosts every rank
    if (first) *first = group ? 0 : ctx->wrank * ctx->per;
    if (count) *count = group ? ctx->n : ctx->per;
  });
}
mics_status mics_set_parallelism(mics_ctx* ctx, int ctas_per_sm, int max_ctas) {
  return guard([&] {
    need(ctx, "ctx");
    if (ctas_per_sm < 0 || max_ctas < 0) mics::raise(MICS_OUT_OF_RANGE, "parallelism must be >= 0");
    each(ctx, [&](mics_ctx* m) {
      m->par_ctas_per_sm = ctas_per_sm;
      m->par_max_ctas = max_ctas;
    });
  });
}
mics_status mics_alloc(mics_ctx* ctx, uint64_t bytes, mics_buf* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    std::vector<mics_buf> b;
    each(ctx, [&](mics_ctx* m) { b.push_back(mics::alloc_sym(m, bytes)); });
    for (const mics_buf& x : b)
      if (x.offset != b[0].offset || x.stride != b[0].stride) mics::raise(MICS_CONFIG_ERROR, "members' arenas diverged");
    *out = b[0];
  });
}
mics_status mics_arena_mark(mics_ctx* ctx, uint64_t* mark) {
  return guard([&] {
    need(ctx, "ctx");
    need(mark, "output");
    *mark = mics::members(ctx)[0]->used;
  });
}
mics_status mics_arena_release(mics_ctx* ctx, uint64_t mark) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) {
      if (mark > m->used) mics::raise(MICS_OUT_OF_RANGE, "mark beyond the arena head");
    });
    each(ctx, [&](mics_ctx* m) {
      MICS_CUDA(cudaStreamSynchronize(m->stream));
      m->used = mark < 4096 ? 4096 : mark;
    });
  });
}
mics_status mics_arena_used(mics_ctx* ctx, uint64_t* used, uint64_t* capacity) {
  return guard([&] {
    need(ctx, "ctx");
    mics_ctx* m = mics::members(ctx)[0];
    if (used) *used = m->used;
    if (capacity) *capacity = m->top;  // what the bump allocator may use
  });
}
mics_status mics_buf_ptr(mics_ctx* ctx, mics_buf buf, int rank, void** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    mics::check_buf_rank(ctx, buf, rank, 0, 0);
    mics_ctx* m = mics::members(ctx)[0];
    if (!m->peer_base[m->process_of(rank)]) mics::raise(MICS_CONFIG_ERROR, "peer arena not imported");
    *out = m->rank_ptr(buf, rank);
  });
}
mics_status mics_memset(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, int value, uint64_t bytes) {
  return guard([&] {
    need(ctx, "ctx");
    mics::check_buf_rank(ctx, buf, rank, off, bytes);
    mics_ctx* m = at_rank(ctx, rank);
    if (!m->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "memset of a rank hosted by another process");
    MICS_CUDA(cudaMemsetAsync(m->rank_ptr(buf, rank) + off, value, bytes, m->stream));
  });
}
mics_status mics_h2d(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, const void* host, uint64_t bytes) {
  return guard([&] {
    need(ctx, "ctx");
    mics::check_buf_rank(ctx, buf, rank, off, bytes);
    mics_ctx* m = at_rank(ctx, rank);
    if (!m->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "h2d into a rank hosted by another process");
    if (bytes) {
      need(host, "host buffer");
      MICS_CUDA(cudaMemcpyAsync(m->rank_ptr(buf, rank) + off, host, bytes, cudaMemcpyHostToDevice, m->stream));
    }
  });
}
mics_status mics_d2h(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, void* host, uint64_t bytes) {
  return guard([&] {
    need(ctx, "ctx");
    mics::check_buf_rank(ctx, buf, rank, off, bytes);
    mics_ctx* m = at_rank(ctx, rank);
    if (!m->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "d2h from a rank hosted by another process");
    if (bytes) {
      need(host, "host buffer");
      MICS_CUDA(cudaMemcpyAsync(host, m->rank_ptr(buf, rank) + off, bytes, cudaMemcpyDeviceToHost, m->stream));
      MICS_CUDA(cudaStreamSynchronize(m->stream));
    }
  });
}
mics_status mics_stream(mics_ctx* ctx, void** s) {
  return guard([&] {
    need(ctx, "ctx");
    need(s, "output");
    *s = mics::members(ctx)[0]->stream;  // a group: its first GPU's stream
  });
}
mics_status mics_synchronize(mics_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { MICS_CUDA(cudaStreamSynchronize(m->stream)); });
  });
}
mics_status mics_barrier(mics_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { mics::barrier_all(m); });
  });
}
mics_status mics_launch_count(mics_ctx* ctx, uint64_t* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    uint64_t n = 0;
    for (mics_ctx* m : mics::members(ctx)) n += m->launches;
    *out = n;
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
    for (mics_ctx* m : mics::members(ctx)) m->traffic_on = on != 0;
  });
}
mics_status mics_traffic_clear(mics_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    for (mics_ctx* m : mics::members(ctx)) m->traffic.clear();
  });
}
}  // extern "C"
namespace {
// a group's members each log the messages their own ranks receive: the union is the log
std::map<std::pair<int, int>, uint64_t> traffic_of(mics_ctx* ctx) {
  if (ctx->subs.empty()) return ctx->traffic;
  std::map<std::pair<int, int>, uint64_t> t;
  for (mics_ctx* m : ctx->subs)
    for (const auto& [k, v] : m->traffic) t[k] += v;
  return t;
}
}  // namespace
extern "C" {
mics_status mics_traffic_size(mics_ctx* ctx, uint64_t* entries) {
  return guard([&] {
    need(ctx, "ctx");
    need(entries, "output");
    *entries = traffic_of(ctx).size();
  });
}
mics_status mics_traffic_get(mics_ctx* ctx, int64_t* t, uint64_t cap) {
  return guard([&] {
    need(ctx, "ctx");
    uint64_t i = 0;
    for (const auto& [key, bytes] : traffic_of(ctx)) {
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
    each(ctx, [&](mics_ctx* m) { mics::all_gather(m, ranks, p, d_shard, chunk, d_out); });
  });
}
mics_status mics_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* d_in, uint64_t in_elems,
                                uint64_t valid, mics_dtype in_t, mics_dtype acc_t, double scale, mics_rs_mode mode,
                                void* const* d_out) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { mics::reduce_scatter(m, ranks, p, d_in, in_elems, valid, in_t, acc_t, scale, int(mode), d_out); });
  });
}
mics_status mics_all_reduce(mics_ctx* ctx, const int* ranks, int p, void* const* buf, uint64_t elems, mics_dtype dt) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { mics::all_reduce(m, ranks, p, buf, elems, dt); });
  });
}
mics_status mics_hier_all_gather(mics_ctx* ctx, int p, int k, const void* const* d_shard, uint64_t chunk,
                                 void* const* d_out, int corrupt) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { mics::hier_all_gather(m, m->n, p, k, d_shard, chunk, d_out, corrupt); });
  });
}
mics_status mics_batched_all_gather(mics_ctx* ctx, const mics_ag_desc* d, int count) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { mics::batched_all_gather(m, d, count); });
  });
}
mics_status mics_batched_reduce_scatter(mics_ctx* ctx, const mics_rs_desc* d, int count, mics_dtype in_t,
                                        mics_dtype acc_t, double scale, mics_rs_mode mode) {
  return guard([&] {
    need(ctx, "ctx");
    each(ctx, [&](mics_ctx* m) { mics::batched_reduce_scatter(m, d, count, in_t, acc_t, scale, int(mode)); });
  });
}
mics_status mics_plan_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* d_shard, uint64_t chunk,
                                 void* const* d_out, mics_plan** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = make_plan(ctx, [&](mics_ctx* m) { return mics::build_all_gather(m, ranks, p, d_shard, chunk, d_out, true); });
  });
}
mics_status mics_plan_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* d_in,
                                     uint64_t in_elems, uint64_t valid, mics_dtype in_t, mics_dtype acc_t,
                                     double scale, mics_rs_mode mode, void* const* d_out, mics_plan** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    *out = make_plan(ctx, [&](mics_ctx* m) {
      return mics::build_reduce_scatter(m, ranks, p, d_in, in_elems, valid, in_t, acc_t, scale, int(mode), d_out,
                                        true);
    });
  });
}
mics_status mics_plan_run(mics_ctx* ctx, mics_plan* plan, int iterations) {
  return guard([&] {
    need(ctx, "ctx");
    need(plan, "plan");
    for (int i = 0; i < iterations; ++i)
      for (const auto& [m, l] : plan->launches) {
        MICS_CUDA(cudaSetDevice(m->device));
        mics::enqueue(m, l);
      }
  });
}
mics_status mics_plan_destroy(mics_plan* plan) {
  return guard([&] {
    if (!plan) return;
    for (auto& [m, l] : plan->launches) {
      cudaSetDevice(m->device);
      l.release();
    }
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
}  // extern "C"
namespace {
mics_sync* sync0(mics_sync* st) { return st->subs.empty() ? st : st->subs[0]; }
// f(member state) for every member (the state itself when it is not a group's)
template <typename F>
void each_sync(mics_sync* st, F&& f) {
  if (st->subs.empty()) {
    f(st);
    return;
  }
  for (mics_sync* m : st->subs) {
    MICS_CUDA(cudaSetDevice(m->ctx->device));
    f(m);
  }
}
}  // namespace
extern "C" {
mics_status mics_sync_create(mics_ctx* ctx, int p, int s, int nseg, const uint64_t* seg_len, mics_dtype acc_t,
                             uint32_t align, mics_sync** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    if (ctx->subs.empty()) {
      *out = mics::sync_create(ctx, p, s, nseg, seg_len, acc_t, align);
      return;
    }
    auto* g = new mics_sync();
    try {
      each(ctx, [&](mics_ctx* m) { g->subs.push_back(mics::sync_create(m, p, s, nseg, seg_len, acc_t, align)); });
    } catch (...) {
      for (mics_sync* m : g->subs) delete m;
      delete g;
      throw;
    }
    *out = g;
  });
}
mics_status mics_sync_destroy(mics_sync* st) {
  return guard([&] {
    if (st)
      for (mics_sync* m : st->subs) delete m;
    delete st;
  });
}
mics_status mics_sync_get_info(mics_sync* st, mics_sync_info* info) {
  return guard([&] {
    need(st, "sync");
    need(info, "output");
    st = sync0(st);
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
    st = sync0(st);
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
    each_sync(st, [&](mics_sync* m) { mics::micro_step(m, grads, off, grad_t, scale, int(mode)); });
  });
}
mics_status mics_sync_boundary(mics_ctx* ctx, mics_sync* st, const mics_adam* adam) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    each_sync(st, [&](mics_sync* m) { mics::boundary(m, adam); });
  });
}
mics_status mics_sync_alt_step(mics_ctx* ctx, mics_sync* st, mics_buf grads, uint64_t off, mics_dtype grad_t,
                               double scale) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    each_sync(st, [&](mics_sync* m) { mics::alt_step(m, grads, off, grad_t, scale); });
  });
}
mics_status mics_sync_alt_boundary(mics_ctx* ctx, mics_sync* st) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "sync");
    each_sync(st, [&](mics_sync* m) { mics::alt_boundary(m); });
  });
}
mics_status mics_sync_events(mics_sync* st, int64_t* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    need(st, "sync");
    st = sync0(st);
    if (count) *count = st->events.size();
    for (uint64_t i = 0; i < st->events.size() && i < cap; ++i)
      for (int k = 0; k < 4; ++k) out[4 * i + uint64_t(k)] = st->events[i][size_t(k)];
  });
}
mics_status mics_sync_clear_events(mics_sync* st) {
  return guard([&] {
    need(st, "sync");
    each_sync(st, [&](mics_sync* m) { m->events.clear(); });
  });
}

// ---- generator
mics_status mics_generate(mics_ctx* ctx, mics_buf buf, int rank, uint64_t off, mics_dtype dt, uint64_t seed, int step,
                          int layer, uint64_t start, uint64_t count) {
  return guard([&] {
    need(ctx, "ctx");
    if (dt != MICS_F32 && dt != MICS_BF16) mics::raise(MICS_TYPE_MISMATCH, "generator emits f32 or bf16");
    mics::check_buf_rank(ctx, buf, rank, off, count * mics::dtype_size(dt));
    mics_ctx* m = at_rank(ctx, rank);
    if (!m->local(rank)) mics::raise(MICS_OUT_OF_RANGE, "generate into a rank hosted by another process");
    mics::launch_generate(m->stream, m->rank_ptr(buf, rank) + off, dt, seed, rank, step, layer, start, count,
                          m->nsm * 8);
    m->launches++;
  });
}

// ---- step driver
}  // extern "C"
namespace {
template <typename F>
void each_step(mics_step* st, F&& f) {
  if (st->subs.empty()) {
    f(st);
    return;
  }
  for (mics_step* m : st->subs) {
    MICS_CUDA(cudaSetDevice(m->ctx->device));
    f(m);
  }
}
mics_step* step0(mics_step* st) { return st->subs.empty() ? st : st->subs[0]; }
}  // namespace
extern "C" {
mics_status mics_step_create(mics_ctx* ctx, const mics_step_cfg* cfg, mics_step** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "output");
    if (ctx->subs.empty()) {
      *out = mics::step_create(ctx, cfg);
      return;
    }
    // members plan their ranks' share; then every member's initial parameters are
    // written (stream sync) before any member gathers them (device barrier)
    auto* g = new mics_step();
    try {
      each(ctx, [&](mics_ctx* m) { g->subs.push_back(mics::step_create(m, cfg, false)); });
      each(ctx, [&](mics_ctx* m) { MICS_CUDA(cudaStreamSynchronize(m->stream)); });
      each(ctx, [&](mics_ctx* m) { mics::barrier_all(m); });
      each(ctx, [&](mics_ctx* m) { MICS_CUDA(cudaStreamSynchronize(m->stream)); });
      g->gsync = new mics_sync();
      for (mics_step* m : g->subs) g->gsync->subs.push_back(m->sync);
      g->ctx = ctx;
    } catch (...) {
      for (mics_step* m : g->subs) mics::step_destroy(m);
      delete g;
      throw;
    }
    *out = g;
  });
}
mics_status mics_step_destroy(mics_step* st) {
  return guard([&] {
    if (st && !st->subs.empty()) {
      for (mics_step* m : st->subs) {
        cudaSetDevice(m->ctx->device);
        mics::step_destroy(m);
      }
      st->gsync->subs.clear();  // the member states died with the member steps
      delete st->gsync;
      delete st;
      return;
    }
    mics::step_destroy(st);
  });
}
mics_status mics_step_run(mics_ctx* ctx, mics_step* st, int iters) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    each_step(st, [&](mics_step* m) { mics::step_run(m, iters); });
  });
}
mics_status mics_step_stats_get(mics_step* st, mics_step_stats* out) {
  return guard([&] {
    need(st, "step");
    need(out, "output");
    *out = step0(st)->stats;  // per GPU (a group's members are alike)
  });
}
mics_status mics_step_sync(mics_step* st, mics_sync** out) {
  return guard([&] {
    need(st, "step");
    need(out, "output");
    *out = st->subs.empty() ? st->sync : st->gsync;
  });
}
mics_status mics_step_buffers(mics_step* st, mics_buf* pb, mics_buf* master, mics_buf* m, mics_buf* v, mics_buf* g,
                              mics_buf* grads) {
  return guard([&] {
    need(st, "step");
    st = step0(st);
    if (pb) *pb = st->pbf16;
    if (master) *master = st->master;
    if (m) *m = st->m;
    if (v) *v = st->v;
    if (g) *g = st->gathered;
    if (grads) *grads = st->grads;
  });
}
}  // extern "C"
namespace {
// every member enqueues its profiled step before any waits for its events (their
// kernels meet at device barriers); per phase, the slowest member
void profile_all(mics_step* st, double* ms) {
  if (st->subs.empty()) {
    mics::step_profile(st, ms);
    return;
  }
  std::vector<mics::ProfileRec*> recs;
  each_step(st, [&](mics_step* m) { recs.push_back(mics::step_profile_begin(m)); });
  for (int i = 0; i < 5; ++i) ms[i] = 0;
  for (size_t d = 0; d < st->subs.size(); ++d) {
    double x[5];
    MICS_CUDA(cudaSetDevice(st->subs[d]->ctx->device));
    mics::step_profile_end(st->subs[d], recs[d], x);
    for (int i = 0; i < 5; ++i) ms[i] = std::max(ms[i], x[i]);
  }
}
}  // namespace
extern "C" {
mics_status mics_step_profile(mics_ctx* ctx, mics_step* st, double* ag, double* rs, double* bnd, double* gen) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    double ms[5];
    profile_all(st, ms);
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
    profile_all(st, ms5);
  });
}
mics_status mics_step_run_host(mics_ctx* ctx, mics_step* st, const void* host_grads, int iters, void* host_result) {
  return guard([&] {
    need(ctx, "ctx");
    need(st, "step");
    need(host_grads, "host gradients");
    // a group's members write their ranks' result slices at their ranks' positions
    uint64_t at = 0;
    each_step(st, [&](mics_step* m) {
      const uint64_t rb = std::min(m->host_result_elems, m->sync->shard_elems) * 4;
      mics::step_run_host(m, host_grads, iters, host_result ? static_cast<char*>(host_result) + at : nullptr);
      at += uint64_t(m->ctx->per) * rb;
    });
  });
}

}  // extern "C"

mics_status mics_gemm_bf16(mics_ctx* ctx, const void* a, uint64_t lda, int a_mn, const void* b, uint64_t ldb, int b_mn,
                           void* c, uint64_t ldc, mics_dtype c_t, int m, int n, int k, int accumulate) {
  return guard([&] {
    need(ctx, "ctx");
    if (!a || !b || !c) mics::raise(MICS_OUT_OF_RANGE, "gemm: null operand");
    mics_ctx* x = mics::members(ctx)[0];  // a group: its first GPU
    MICS_CUDA(cudaSetDevice(x->device));
    const mics::GemmLaunch g = mics::plan_gemm(a, lda, a_mn, b, ldb, b_mn, c, ldc, c_t, m, n, k, accumulate);
    mics::launch_gemm(x->stream, g);
    x->launches++;
  });
}
