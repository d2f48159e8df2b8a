// Collective planners: turn the reference's collective calls into descriptor
// tables for the sm_100a pull engines (kernels.cu) and enqueue them.
//
//   all_gather              collectives.cpp:103-134  -> one k_copy launch
//   reduce_scatter          collectives.cpp:136-183  -> one k_reduce launch
//   all_reduce              collectives.cpp:185-190  -> k_reduce (in place) + k_copy
//   hierarchical_all_gather collectives.cpp:192-291  -> two k_copy launches
//   batched_*               collectives.cpp:293-321  -> one launch for the whole batch
//
// Traffic is recorded with the reference's own per-message accounting
// (record_traffic calls at collectives.cpp:120, :162 and inside the stages), so
// mics_traffic_get() equals VirtualRankEngine::traffic() for the same calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "internal.h"

namespace mics {

void CopyPlan::add(const void* src, const std::vector<void*>& dsts, uint64_t bytes) {
  if (bytes == 0 || dsts.empty()) return;
  for (size_t b = 0; b < dsts.size(); b += kMaxDst) {
    CopySeg s;
    std::memset(&s, 0, sizeof(s));
    s.src = static_cast<const uint8_t*>(src);
    s.bytes = bytes;
    s.ndst = uint32_t(std::min<size_t>(kMaxDst, dsts.size() - b));
    for (uint32_t d = 0; d < s.ndst; ++d) s.dst[d] = static_cast<uint8_t*>(dsts[b + d]);
    s.tile0 = tiles;
    s.gsize = 1;
    tiles += uint32_t(ceil_div(bytes, kCopyTile));
    segs.push_back(s);
  }
}

void CopyPlan::add_group(const std::vector<std::pair<const void*, std::vector<void*>>>& items, uint64_t bytes) {
  if (bytes == 0) return;
  const size_t first = segs.size();
  const uint32_t t0 = tiles;
  for (const auto& it : items) add(it.first, it.second, bytes);
  const uint32_t k = uint32_t(segs.size() - first);
  if (k <= 1) return;
  for (size_t i = first; i < segs.size(); ++i) {  // one interleaved tile range for the whole group
    segs[i].tile0 = t0;
    segs[i].gsize = k;
  }
  tiles = t0 + k * uint32_t(ceil_div(bytes, kCopyTile));
}

void HierPlan::add_group(int stage, const std::vector<std::tuple<const void*, void*, uint64_t*>>& items,
                         uint64_t bytes, int lag) {
  if (bytes == 0 || items.empty()) return;
  const uint32_t t0 = tiles, per = uint32_t(ceil_div(bytes, kCopyTile)), k = uint32_t(items.size());
  for (const auto& [s, d, f] : items) {
    HierSeg g;
    std::memset(&g, 0, sizeof(g));
    g.src = static_cast<const uint8_t*>(s);
    g.dst = static_cast<uint8_t*>(d);
    g.flags = f;
    g.bytes = bytes;
    g.tile0 = t0;
    g.gsize = k;
    g.stage = uint32_t(stage);
    g.lag = uint32_t(lag);
    segs.push_back(g);
  }
  tiles = t0 + k * per;
}

// Stage 1 (collectives.cpp:229-241): rank r = base + m*k + j gathers channel j's chunks
// from the q ranks base + m2*k + j, stage 2 (:243-265) folded into the store position
// (m2*k + j, or j*q + m2 with corrupt_stage2); stage 3 (:267-288): r pulls positions
// t*k + j2 (corrupt: j2*q + t) from each node peer base + m*k + j2, j2 != j — the
// peer's stage-1 chunk t, guarded by that chunk's tile flags.
HierPlan plan_hier(mics_ctx* ctx, int n, int p, int k, uint64_t chunk, int corrupt,
                   const std::function<const void*(int)>& src, const std::function<char*(int, uint64_t)>& dst,
                   const std::function<uint64_t*(int)>& flags, uint64_t ftiles, int stages, int lag) {
  HierPlan plan;
  const int q = p / k;
  using Item = std::tuple<const void*, void*, uint64_t*>;
  std::vector<std::vector<Item>> st3;
  for (int g = 0; g < n / p; ++g) {
    const int base = g * p;
    for (int m = 0; m < q; ++m)
      for (int j = 0; j < k; ++j) {
        const int r = base + m * k + j;
        if (!ctx->local(r)) continue;
        std::vector<Item> s1, s3;
        for (int j2 = 0; j2 < k; ++j2)  // a node peer elsewhere reads / publishes flags across GPUs
          if (j2 != j) plan.sys |= !ctx->local(base + m * k + j2);
        for (int m2 = 0; m2 < q && (stages & 1); ++m2) {
          const uint64_t pos = corrupt ? uint64_t(j) * q + m2 : uint64_t(m2) * k + j;
          const int from = base + m2 * k + j;
          s1.emplace_back(src(from), dst(r, pos), flags(r) + uint64_t(m2) * ftiles);
          (ctx->local(from) ? plan.hbm_bytes : plan.remote_bytes) += chunk;
          plan.hbm_bytes += chunk;
        }
        for (int j2 = 0; j2 < k && (stages & 2); ++j2) {
          if (j2 == j) continue;
          const int from = base + m * k + j2;
          for (int t = 0; t < q; ++t) {
            const uint64_t pos = corrupt ? uint64_t(j2) * q + t : uint64_t(t) * k + j2;
            s3.emplace_back(dst(from, pos), dst(r, pos), flags(from) + uint64_t(t) * ftiles);
            (ctx->local(from) ? plan.hbm_bytes : plan.remote_bytes) += chunk;
            plan.hbm_bytes += chunk;
          }
        }
        plan.add_group(1, s1, chunk);
        st3.push_back(std::move(s3));
      }
  }
  for (const auto& s3 : st3) plan.add_group(3, s3, chunk, lag);  // every stage-1 tile precedes every stage-3 tile
  return plan;
}

HierPlan concat_hier(const HierPlan& a, const HierPlan& b) {
  HierPlan c = a;
  for (HierSeg g : b.segs) {
    g.tile0 += a.tiles;
    c.segs.push_back(g);
  }
  c.tiles = a.tiles + b.tiles;
  c.sys = a.sys || b.sys;
  c.remote_bytes += b.remote_bytes;
  c.hbm_bytes += b.hbm_bytes;
  return c;
}

void RedPlan::add(const std::vector<const void*>& src, void* dst, uint64_t elems, uint64_t valid) {
  if (elems == 0) return;
  RedJob j;
  std::memset(&j, 0, sizeof(j));
  j.dst = static_cast<uint8_t*>(dst);
  j.elems = elems;
  j.valid = std::min(valid, elems);
  j.p = uint32_t(src.size());
  j.tile0 = tiles;
  max_p = std::max(max_p, j.p);
  uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  for (const void* s : src) a |= reinterpret_cast<uintptr_t>(s);
  j.aligned = (a & 15) == 0;
  tiles += uint32_t(ceil_div(elems, tile_elems));
  jobs.push_back(j);
  srcs.push_back(src);
}

void AdamPlan::add(const std::vector<const void*>& src, float* param, float* m, float* v, uint16_t* pbf16, float* gout,
                   uint64_t elems, uint64_t sub) {
  if (elems == 0) return;
  AdamJob j;
  std::memset(&j, 0, sizeof(j));
  j.param = param;
  j.m = m;
  j.v = v;
  j.pbf16 = pbf16;
  j.gout = gout;
  j.elems = elems;
  j.sub = sub;
  j.rr = uint32_t(src.size());
  j.tile0 = tiles;
  tiles += uint32_t(src.size() * ceil_div(sub, kAdamTile));  // rr slices, tiles interleaved (k_adam)
  jobs.push_back(j);
  srcs.push_back(src);
}

void AdamPlan::add_replica(float* param2, float* m2, float* v2, uint16_t* pbf16_2) {
  AdamJob& j = jobs.back();
  j.param2 = param2;
  j.m2 = m2;
  j.v2 = v2;
  j.pbf16_2 = pbf16_2;
}

void Launch::release() {
  if (d_desc) cudaFree(d_desc);
  d_desc = nullptr;
}

namespace {
void* table_memory(mics_ctx* ctx, uint64_t bytes, bool persistent) {
  if (!persistent) return ctx->ring_reserve(bytes);
  void* d = nullptr;
  MICS_CUDA(cudaMalloc(&d, bytes ? bytes : 16));
  return d;
}
void table_upload(mics_ctx* ctx, void* d, const void* h, uint64_t bytes, bool persistent) {
  if (persistent)
    MICS_CUDA(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  else
    ctx->ring_upload(d, h, bytes);
}

// jobs followed by their source-pointer arrays, pointers patched to device addresses
template <typename Job>
void* upload_jobs(mics_ctx* ctx, std::vector<Job> jobs, const std::vector<std::vector<const void*>>& srcs,
                  bool persistent, uint64_t* table_bytes = nullptr) {
  uint64_t nptr = 0;
  for (const auto& s : srcs) nptr += s.size();
  const uint64_t jbytes = round_up(sizeof(Job) * jobs.size(), 16);
  const uint64_t bytes = round_up(jbytes + nptr * sizeof(void*), 16);
  if (table_bytes) *table_bytes = bytes;
  char* d = static_cast<char*>(table_memory(ctx, bytes, persistent));
  std::vector<char> blob(bytes);
  const void** ptrs = reinterpret_cast<const void**>(blob.data() + jbytes);
  uint64_t k = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    using P = decltype(jobs[i].srcs);
    jobs[i].srcs = reinterpret_cast<P>(d + jbytes + k * sizeof(void*));
    for (const void* s : srcs[i]) ptrs[k++] = s;
  }
  std::memcpy(blob.data(), jobs.data(), sizeof(Job) * jobs.size());
  table_upload(ctx, d, blob.data(), bytes, persistent);
  return d;
}
}  // namespace

Launch make_copy_launch(mics_ctx* ctx, const CopyPlan& plan, const BarrierArg& bar, bool persistent) {
  Launch l;
  l.kind = Launch::COPY;
  l.ndesc = int(plan.segs.size());
  l.ntiles = plan.tiles;
  l.grid = ctx->grid_for(plan.tiles, ctx->occ_copy);
  l.bar = bar;
  for (const auto& s : plan.segs) {
    (ctx->is_local_ptr(s.src) ? l.hbm_bytes : l.remote_bytes) += s.bytes;
    l.hbm_bytes += s.bytes * s.ndst;
  }
  if (l.ndesc) {
    const uint64_t bytes = sizeof(CopySeg) * plan.segs.size();
    l.d_desc = table_memory(ctx, bytes, persistent);
    table_upload(ctx, l.d_desc, plan.segs.data(), bytes, persistent);
  }
  return l;
}

Launch make_hier_launch(mics_ctx* ctx, const HierPlan& plan, const BarrierArg& bar, int chan, bool persistent) {
  Launch l;
  l.kind = Launch::HIER;
  l.ndesc = int(plan.segs.size());
  l.ntiles = plan.tiles;
  // one resident wave: stage-3 tiles wait for stage-1 tiles of other CTAs
  l.grid = ctx->grid_for(plan.tiles, ctx->occ_hier);
  l.bar = bar;
  l.hier_sys = plan.sys ? 1 : 0;
  l.hier_chan = chan;
  l.remote_bytes = plan.remote_bytes;
  l.hbm_bytes = plan.hbm_bytes;
  if (l.ndesc) {
    const uint64_t bytes = sizeof(HierSeg) * plan.segs.size();
    l.d_desc = table_memory(ctx, bytes, persistent);
    table_upload(ctx, l.d_desc, plan.segs.data(), bytes, persistent);
  }
  return l;
}

Launch make_reduce_launch(mics_ctx* ctx, const RedPlan& plan, mics_dtype in_t, mics_dtype acc_t, double scale,
                          int mode, const BarrierArg& bar, bool persistent) {
  Launch l;
  l.kind = Launch::REDUCE;
  l.ndesc = int(plan.jobs.size());
  l.ntiles = plan.tiles;
  l.grid = ctx->grid_for(plan.tiles, ctx->reduce_occ(in_t, plan.max_p));
  l.max_p = plan.max_p;
  l.in_t = in_t;
  l.acc_t = acc_t;
  l.scale = scale;
  l.mode = mode;
  l.bar = bar;
  const uint64_t szi = dtype_size(in_t), sza = dtype_size(acc_t);
  for (size_t j = 0; j < plan.jobs.size(); ++j) {
    const RedJob& J = plan.jobs[j];
    for (const void* s : plan.srcs[j]) (ctx->is_local_ptr(s) ? l.hbm_bytes : l.remote_bytes) += J.valid * szi;
    l.hbm_bytes += J.elems * sza * (mode == MICS_RS_ACCUMULATE ? 2 : 1);
  }
  if (l.ndesc) l.d_desc = upload_jobs(ctx, plan.jobs, plan.srcs, persistent, &l.table_bytes);
  return l;
}

Launch make_adam_launch(mics_ctx* ctx, const AdamPlan& plan, const AdamScalars& sc, const BarrierArg& bar,
                        bool persistent) {
  Launch l;
  l.kind = Launch::ADAM;
  l.ndesc = int(plan.jobs.size());
  l.ntiles = plan.tiles;
  l.grid = ctx->grid_for(plan.tiles, ctx->occ_adam);
  l.adam = sc;
  l.bar = bar;
  for (size_t j = 0; j < plan.jobs.size(); ++j) {
    const AdamJob& J = plan.jobs[j];
    for (size_t q = 0; q < plan.srcs[j].size(); ++q) {  // owner q holds slice [q*sub, (q+1)*sub)
      const uint64_t lo = std::min<uint64_t>(q * J.sub, J.elems), hi = std::min<uint64_t>((q + 1) * J.sub, J.elems);
      (ctx->is_local_ptr(plan.srcs[j][q]) ? l.hbm_bytes : l.remote_bytes) += (hi - lo) * 4;
    }
    l.hbm_bytes += J.elems * (24 + (J.pbf16 ? 2 : 0) + (J.gout ? 4 : 0));  // r/w p, m, v; w bf16; w grad
    if (J.param2) l.hbm_bytes += J.elems * (24 + (J.pbf16_2 ? 2 : 0));      // the second replica's state
  }
  if (l.ndesc) l.d_desc = upload_jobs(ctx, plan.jobs, plan.srcs, persistent);
  return l;
}

void enqueue(mics_ctx* ctx, const Launch& l, int dep_first, cudaStream_t stream) {
  cudaStream_t st = stream ? stream : ctx->stream;
  // A launch without local work still runs (one CTA) when it carries a barrier:
  // the peers count on this process's signals.
  if (l.ndesc == 0 && l.bar.mask == 0) return;
  BarrierArg bar = l.bar;
  if (dep_first >= 0) bar.dep_first = dep_first;
  if (bar.mask) bar.dep_first = 1;  // barrier tickets: never overlap the predecessor
  switch (l.kind) {
    case Launch::COPY:
      launch_copy(st, static_cast<const CopySeg*>(l.d_desc), l.ndesc, l.ntiles, l.grid, bar);
      break;
    case Launch::REDUCE:
      launch_reduce(st, l.in_t, l.acc_t, static_cast<const RedJob*>(l.d_desc), l.ndesc, l.table_bytes,
                    l.max_p, l.ntiles, l.grid, l.scale, l.mode, bar);
      break;
    case Launch::ADAM:
      launch_adam(st, static_cast<const AdamJob*>(l.d_desc), l.ndesc, l.ntiles, l.grid, l.adam, l.dyn, bar);
      break;
    case Launch::BARRIER:
      launch_barrier(st, bar);
      break;
    case Launch::HIER: {
      HierArg ha;
      ha.ctl = ctx->d_hctl + l.hier_chan;
      ha.tab = ctx->d_tab + l.hier_chan;
      ha.my_done = l.hier_merged ? reinterpret_cast<uint64_t*>(ctx->base + kDoneOffset) + l.hier_chan : nullptr;
      ha.peer_mask = l.hier_peers;
      ha.sys_scope = l.hier_sys;
      ha.tile_flags = l.hier_merged ? 0 : 1;
      ha.interleave_n1 = l.hier_merged ? l.hier_n1 : 0;
      launch_hier(st, static_cast<const HierSeg*>(l.d_desc), l.ndesc, l.ntiles, l.grid, ha, bar);
      break;
    }
    case Launch::FBND: {
      FbArg a = l.fb;
      a.items = l.ntiles;
      a.sys_scope = l.hier_sys;
      launch_fbnd(st, a, l.grid, l.adam, l.dyn, l.fb_epoch, bar);
      break;
    }
    case Launch::TAIL:
      launch_tail(st, l.in_t, l.tail_r, l.tail_p, static_cast<const TailJob*>(l.d_desc), l.ndesc, l.ntiles, l.grid,
                  l.adam, l.dyn, l.mode, bar);
      break;
  }
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// collectives on device pointers
namespace {

void check_ptrs(const void* const* a, int count, const mics_ctx* ctx, const int* ranks, bool only_local,
                const char* what) {
  if (count > 0 && !a) raise(MICS_OUT_OF_RANGE, std::string(what) + ": null pointer array");
  for (int i = 0; i < count; ++i)
    if (!a[i] && (!only_local || ctx->local(ranks[i])))
      raise(MICS_OUT_OF_RANGE, std::string(what) + ": null buffer at position " + std::to_string(i));
}

void check_rs_types(mics_dtype in_t, mics_dtype acc_t) {
  const bool ok = (in_t == acc_t && in_t != MICS_BF16) || (in_t == MICS_BF16 && acc_t == MICS_F32);
  if (!ok) raise(MICS_TYPE_MISMATCH, "reduce: accumulate type must equal the input type (or f32 for bf16 input)");
}

void plan_all_gather(mics_ctx* ctx, CopyPlan& plan, const int* ranks, int p, const void* const* shard, uint64_t chunk,
                     void* const* out) {
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      if (j != i) ctx->record(ranks[i], ranks[j], chunk);  // collectives.cpp:116-123
  std::vector<int> loc;
  for (int j = 0; j < p; ++j)
    if (ctx->local(ranks[j])) loc.push_back(j);
  if (loc.empty()) return;
  // one read of chunk i feeds every local destination; the p chunks form one
  // stripe group so all sources (NVLink peers and local HBM) stream concurrently
  std::vector<std::pair<const void*, std::vector<void*>>> items;
  for (int i = 0; i < p; ++i) {
    std::vector<void*> dsts;
    for (int j : loc) dsts.push_back(static_cast<char*>(out[j]) + uint64_t(i) * chunk);
    items.emplace_back(shard[i], std::move(dsts));
  }
  plan.add_group(items, chunk);
}

void plan_reduce_scatter(mics_ctx* ctx, RedPlan& plan, const int* ranks, int p, const void* const* in,
                         uint64_t in_elems, uint64_t valid, mics_dtype in_t, void* const* out) {
  const uint64_t chunk = in_elems / uint64_t(p);
  const uint64_t szi = dtype_size(in_t);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      if (j != i) ctx->record(ranks[i], ranks[j], chunk * szi);  // collectives.cpp:157-165
  for (int j = 0; j < p; ++j) {
    if (!ctx->local(ranks[j])) continue;
    std::vector<const void*> srcs(static_cast<size_t>(p));
    for (int i = 0; i < p; ++i) srcs[size_t(i)] = static_cast<const char*>(in[i]) + uint64_t(j) * chunk * szi;
    const uint64_t first = uint64_t(j) * chunk;
    plan.add(srcs, out[j], chunk, valid > first ? valid - first : 0);
  }
}

}  // namespace

Launch build_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* shard, uint64_t chunk,
                        void* const* out, bool persistent) {
  check_group(ctx, ranks, p);
  check_ptrs(shard, p, ctx, ranks, false, "all_gather input");
  check_ptrs(const_cast<const void* const*>(out), p, ctx, ranks, true, "all_gather output");
  CopyPlan plan;
  plan_all_gather(ctx, plan, ranks, p, shard, chunk, out);
  return make_copy_launch(ctx, plan, ctx->barrier(ctx->peer_mask(ranks, p), 1, 1, 0, 0), persistent);
}

void all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* shard, uint64_t chunk, void* const* out) {
  enqueue(ctx, build_all_gather(ctx, ranks, p, shard, chunk, out, false));
}

Launch build_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* in, uint64_t in_elems,
                            uint64_t valid, mics_dtype in_t, mics_dtype acc_t, double scale, int mode,
                            void* const* out, bool persistent) {
  check_group(ctx, ranks, p);
  check_rs_types(in_t, acc_t);
  if (p == 0) return Launch{};
  if (in_elems % uint64_t(p))
    raise(MICS_TYPE_MISMATCH, "reduce_scatter: " + std::to_string(in_elems) + " elements are not divisible into " +
                                  std::to_string(p) + " chunks");  // collectives.cpp:148-153
  if (in_t == MICS_I64 && scale != 1.0) raise(MICS_TYPE_MISMATCH, "reduce_scatter: scale needs a float type");
  check_ptrs(in, p, ctx, ranks, false, "reduce_scatter input");
  check_ptrs(const_cast<const void* const*>(out), p, ctx, ranks, true, "reduce_scatter output");
  RedPlan plan(in_t);
  plan_reduce_scatter(ctx, plan, ranks, p, in, in_elems, valid, in_t, out);
  return make_reduce_launch(ctx, plan, in_t, acc_t, scale, mode, ctx->barrier(ctx->peer_mask(ranks, p), 1, 1, 0, 0),
                            persistent);
}

void reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* in, uint64_t in_elems,
                    uint64_t valid, mics_dtype in_t, mics_dtype acc_t, double scale, int mode, void* const* out) {
  enqueue(ctx, build_reduce_scatter(ctx, ranks, p, in, in_elems, valid, in_t, acc_t, scale, mode, out, false));
}

void all_reduce(mics_ctx* ctx, const int* ranks, int p, void* const* buf, uint64_t elems, mics_dtype dt) {
  check_group(ctx, ranks, p);
  check_rs_types(dt, dt);
  if (p == 0) return;
  if (elems % uint64_t(p))
    raise(MICS_TYPE_MISMATCH, "all_reduce: " + std::to_string(elems) + " elements are not divisible into " +
                                  std::to_string(p) + " chunks");
  check_ptrs(const_cast<const void* const*>(buf), p, ctx, ranks, false, "all_reduce buffer");
  const uint64_t chunk = elems / uint64_t(p), sz = dtype_size(dt), cb = chunk * sz;
  // reduce-scatter in place: position j folds slice j of every buffer into its own slice j
  RedPlan rs(dt);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      if (j != i) ctx->record(ranks[i], ranks[j], cb);
  for (int j = 0; j < p; ++j) {
    if (!ctx->local(ranks[j])) continue;
    std::vector<const void*> srcs(static_cast<size_t>(p));
    for (int i = 0; i < p; ++i) srcs[size_t(i)] = static_cast<const char*>(buf[i]) + uint64_t(j) * cb;
    rs.add(srcs, static_cast<char*>(buf[j]) + uint64_t(j) * cb, chunk, chunk);
  }
  const uint64_t mask = ctx->peer_mask(ranks, p);
  enqueue(ctx, make_reduce_launch(ctx, rs, dt, dt, 1.0, MICS_RS_STORE, ctx->barrier(mask, 1, 1), false));
  // all-gather of the reduced slices
  CopyPlan ag;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      if (j != i) ctx->record(ranks[i], ranks[j], cb);
  std::vector<std::pair<const void*, std::vector<void*>>> items;
  for (int i = 0; i < p; ++i) {
    std::vector<void*> dsts;
    for (int j = 0; j < p; ++j)
      if (j != i && ctx->local(ranks[j])) dsts.push_back(static_cast<char*>(buf[j]) + uint64_t(i) * cb);
    if (!dsts.empty()) items.emplace_back(static_cast<const char*>(buf[i]) + uint64_t(i) * cb, std::move(dsts));
  }
  ag.add_group(items, cb);
  enqueue(ctx, make_copy_launch(ctx, ag, ctx->barrier(mask, 0, 1, 0, 0), false));
}

// Hierarchical all-gather.  For partition group g (base = g*p) with q = p/k
// virtual nodes of k ranks: phase 1 is stage 1 (k channel all-gathers among the
// q ranks sharing a local index) with stage 2's rearrangement folded into the
// store address: C_{m'k+j} lands directly at its final position.  Phase 2 is
// stage 3: every rank pulls from each node peer j' the positions t*k+j'.
// corrupt_stage2 keeps the raw stage-1 layout [C_j, C_{k+j}, ...] at offset
// j*q*chunk and gathers those buffers per node (collectives.cpp:243-257).
// `n` is the cluster's rank count: ctx->n, or (single process) any n <= ctx->n.
void hier_all_gather(mics_ctx* ctx, int n, int p, int k, const void* const* shard, uint64_t chunk,
                     void* const* out, int corrupt) {
  // (a multi-process job plans the whole cluster: n must be the job's rank count)
  if (n < 1 || n > ctx->n || (ctx->world > 1 && !ctx->member && n != ctx->n))
    raise(MICS_SHAPE_ERROR, "cluster has " + std::to_string(n) + " ranks but the context has " +
                                std::to_string(ctx->n));  // collectives.cpp:200-202
  if (p < 1 || p > n)
    raise(MICS_OUT_OF_RANGE, "partition size p=" + std::to_string(p) + " must satisfy 1 <= p <= n=" +
                                 std::to_string(n));
  if (n % p) raise(MICS_NON_DIVISIBLE, "partition size p=" + std::to_string(p) + " does not divide n=" +
                                           std::to_string(n));
  if (k < 1 || n % k) raise(MICS_SHAPE_ERROR, "cluster of k=" + std::to_string(k) + " ranks per node does not tile n=" +
                                                  std::to_string(n));
  if (!mics_partition_shape_ok(p, k))
    raise(MICS_SHAPE_ERROR, "partition size p=" + std::to_string(p) + " is not node-aligned for k=" +
                                std::to_string(k));  // collectives.cpp:208-210
  std::vector<int> all(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) all[size_t(r)] = r;
  check_ptrs(shard, n, ctx, all.data(), false, "hierarchical_all_gather input");
  // phase 2 pulls from node peers' outputs: every entry must be valid (peer-mapped)
  check_ptrs(const_cast<const void* const*>(out), n, ctx, all.data(), p <= k, "hierarchical_all_gather output");

  auto O = [&](int r, uint64_t pos) { return static_cast<char*>(out[r]) + pos * chunk; };
  uint64_t mask = 0;
  if (p <= k) {  // single-node partition group: plain all-gather (collectives.cpp:218-225)
    CopyPlan plan;
    for (int g = 0; g < n / p; ++g) {
      plan_all_gather(ctx, plan, all.data() + g * p, p, shard + g * p, chunk, out + g * p);
      mask |= ctx->peer_mask(all.data() + g * p, p);
    }
    enqueue(ctx, make_copy_launch(ctx, plan, ctx->barrier(mask, 1, 1, 0, 0), false));
    return;
  }
  const int q = p / k;
  for (int g = 0; g < n / p; ++g) {
    const int base = g * p;
    mask |= ctx->peer_mask(all.data() + base, p);
    // traffic of the reference's stages (stage 1 :233-241, stage 3 :267-288 / corrupt :246-255)
    for (int j = 0; j < k; ++j)
      for (int m = 0; m < q; ++m)
        for (int m2 = 0; m2 < q; ++m2)
          if (m2 != m) ctx->record(base + m * k + j, base + m2 * k + j, chunk);
    for (int m = 0; m < q; ++m)
      for (int j = 0; j < k; ++j)
        for (int j2 = 0; j2 < k; ++j2)
          if (j2 != j) ctx->record(base + m * k + j, base + m * k + j2, uint64_t(q) * chunk);
  }
  // one launch: entry barrier (inputs ready everywhere), stage-1 tiles publish flags,
  // stage-3 tiles consume them, exit barrier (done reading the peers' buffers)
  const uint64_t ft = hier_flag_tiles(chunk);
  const mics_buf fb = hier_flags(ctx, uint64_t(q) * ft * 8);
  HierPlan plan = plan_hier(
      ctx, n, p, k, chunk, corrupt, [&](int r) { return shard[r]; }, O,
      [&](int r) { return reinterpret_cast<uint64_t*>(ctx->rank_ptr(fb, r)); }, ft);
  enqueue(ctx, make_hier_launch(ctx, plan, ctx->barrier(mask, 1, 1, 0, 0), 0, false));
}

void batched_all_gather(mics_ctx* ctx, const mics_ag_desc* d, int count) {
  if (count < 0 || (count > 0 && !d)) raise(MICS_OUT_OF_RANGE, "batched_all_gather: bad descriptor list");
  CopyPlan plan;
  uint64_t mask = 0;
  for (int b = 0; b < count; ++b) {
    check_group(ctx, d[b].ranks, d[b].p);
    check_ptrs(d[b].d_shard, d[b].p, ctx, d[b].ranks, false, "batched_all_gather input");
    check_ptrs(const_cast<const void* const*>(d[b].d_out), d[b].p, ctx, d[b].ranks, true, "batched_all_gather output");
    plan_all_gather(ctx, plan, d[b].ranks, d[b].p, d[b].d_shard, d[b].chunk_bytes, d[b].d_out);
    mask |= ctx->peer_mask(d[b].ranks, d[b].p);
  }
  enqueue(ctx, make_copy_launch(ctx, plan, ctx->barrier(mask, 1, 1, 0, 0), false));
}

void batched_reduce_scatter(mics_ctx* ctx, const mics_rs_desc* d, int count, mics_dtype in_t, mics_dtype acc_t,
                            double scale, int mode) {
  if (count < 0 || (count > 0 && !d)) raise(MICS_OUT_OF_RANGE, "batched_reduce_scatter: bad descriptor list");
  check_rs_types(in_t, acc_t);
  RedPlan plan(in_t);
  uint64_t mask = 0;
  for (int b = 0; b < count; ++b) {
    check_group(ctx, d[b].ranks, d[b].p);
    if (d[b].p == 0) continue;
    if (d[b].in_elems % uint64_t(d[b].p))
      raise(MICS_TYPE_MISMATCH, "batched_reduce_scatter: descriptor " + std::to_string(b) +
                                    " is not divisible into whole chunks");
    check_ptrs(d[b].d_in, d[b].p, ctx, d[b].ranks, false, "batched_reduce_scatter input");
    check_ptrs(const_cast<const void* const*>(d[b].d_out), d[b].p, ctx, d[b].ranks, true,
               "batched_reduce_scatter output");
    plan_reduce_scatter(ctx, plan, d[b].ranks, d[b].p, d[b].d_in, d[b].in_elems, d[b].valid_elems, in_t, d[b].d_out);
    mask |= ctx->peer_mask(d[b].ranks, d[b].p);
  }
  enqueue(ctx, make_reduce_launch(ctx, plan, in_t, acc_t, scale, mode, ctx->barrier(mask, 1, 1, 0, 0), false));
}

// ---------------------------------------------------------------------------
// host-buffer drop-ins: stage through the arena, run, copy back.  On a multi-device
// context (mics_init_devices) every member stages the buffers of the ranks it hosts in
// blocks at the same arena offset, runs its part of the collective (pulling the other
// members' blocks over NVLink by UVA pointer) and copies its ranks' results back; the
// members' kernels meet at the device flag barriers.
namespace {
constexpr uint64_t kStage = 256;  // keep every staged buffer 16-byte aligned

class Staging {
 public:
  explicit Staging(mics_ctx* ctx) : ctx_(ctx), mem_(members(ctx)) {
    if (ctx->world != 1 && ctx->subs.empty())
      raise(MICS_CONFIG_ERROR, "host-buffer API needs a single-process context (one GPU, or mics_init_devices)");
    for (mics_ctx* m : mem_) marks_.push_back(m->used);
  }
  ~Staging() {
    for (size_t i = 0; i < mem_.size(); ++i) mem_[i]->used = marks_[i];
  }
  uint64_t block(uint64_t bytes) {  // the same offset in every member (identical allocation sequences)
    const uint64_t off = mem_[0]->local_alloc(bytes);
    for (size_t i = 1; i < mem_.size(); ++i)
      if (mem_[i]->local_alloc(bytes) != off) raise(MICS_CONFIG_ERROR, "members' arenas diverged");
    return off;
  }
  mics_ctx* owner(int rank) const { return mics::owner(ctx_, rank); }
  char* at(uint64_t block, int rank, uint64_t off) const { return owner(rank)->base + block + off; }
  void h2d(int rank, void* dst, const void* src, uint64_t bytes) const {
    if (!bytes) return;
    mics_ctx* m = owner(rank);
    MICS_CUDA(cudaSetDevice(m->device));
    MICS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, m->stream));
  }
  void d2h(int rank, void* dst, const void* src, uint64_t bytes) const {
    if (!bytes) return;
    mics_ctx* m = owner(rank);
    MICS_CUDA(cudaSetDevice(m->device));
    MICS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, m->stream));
  }
  template <typename F>
  void each(F&& f) const {
    for (mics_ctx* m : mem_) {
      MICS_CUDA(cudaSetDevice(m->device));
      f(m);
    }
  }
  void finish() const {
    each([](mics_ctx* m) { MICS_CUDA(cudaStreamSynchronize(m->stream)); });
  }

 private:
  mics_ctx* ctx_;
  std::vector<mics_ctx*> mem_;
  std::vector<uint64_t> marks_;
};
}  // namespace

void host_all_gather(mics_ctx* ctx, const int* ranks, int p, const void* const* shards, uint64_t chunk,
                     void* const* out) {
  check_group(ctx, ranks, p);
  Staging s(ctx);
  const uint64_t cs = round_up(chunk, kStage), os = round_up(uint64_t(p) * chunk, kStage);
  const uint64_t in = s.block(cs * uint64_t(p)), ob = s.block(os * uint64_t(p));
  std::vector<const void*> ip(static_cast<size_t>(p));
  std::vector<void*> op(static_cast<size_t>(p));
  for (int i = 0; i < p; ++i) {
    ip[size_t(i)] = s.at(in, ranks[i], uint64_t(i) * cs);
    op[size_t(i)] = s.at(ob, ranks[i], uint64_t(i) * os);
    s.h2d(ranks[i], const_cast<void*>(ip[size_t(i)]), shards[i], chunk);
  }
  s.each([&](mics_ctx* m) { all_gather(m, ranks, p, ip.data(), chunk, op.data()); });
  for (int j = 0; j < p; ++j) s.d2h(ranks[j], out[j], op[size_t(j)], uint64_t(p) * chunk);
  s.finish();
}

void host_reduce_scatter(mics_ctx* ctx, const int* ranks, int p, const void* const* bufs, uint64_t bytes,
                         mics_dtype dt, void* const* out) {
  check_group(ctx, ranks, p);
  Staging s(ctx);
  if (dt == MICS_BF16) raise(MICS_TYPE_MISMATCH, "reduce_scatter: bf16 is not a reduction type");
  if (p == 0) return;
  const uint64_t sz = dtype_size(dt);
  if (bytes % (uint64_t(p) * sz))
    raise(MICS_TYPE_MISMATCH, "reduce_scatter: buffer of " + std::to_string(bytes) + " bytes is not divisible into " +
                                  std::to_string(p) + " chunks of whole " + std::to_string(sz) + "-byte elements");
  const uint64_t bs = round_up(bytes, kStage), cb = bytes / uint64_t(p), cs = round_up(cb, kStage);
  const uint64_t in = s.block(bs * uint64_t(p)), ob = s.block(cs * uint64_t(p));
  std::vector<const void*> ip(static_cast<size_t>(p));
  std::vector<void*> op(static_cast<size_t>(p));
  for (int i = 0; i < p; ++i) {
    ip[size_t(i)] = s.at(in, ranks[i], uint64_t(i) * bs);
    op[size_t(i)] = s.at(ob, ranks[i], uint64_t(i) * cs);
    s.h2d(ranks[i], const_cast<void*>(ip[size_t(i)]), bufs[i], bytes);
  }
  s.each([&](mics_ctx* m) {
    reduce_scatter(m, ranks, p, ip.data(), bytes / sz, bytes / sz, dt, dt, 1.0, MICS_RS_STORE, op.data());
  });
  for (int j = 0; j < p; ++j) s.d2h(ranks[j], out[j], op[size_t(j)], cb);
  s.finish();
}

void host_all_reduce(mics_ctx* ctx, const int* ranks, int p, const void* const* bufs, uint64_t bytes, mics_dtype dt,
                     void* const* out) {
  check_group(ctx, ranks, p);
  Staging s(ctx);
  if (dt == MICS_BF16) raise(MICS_TYPE_MISMATCH, "all_reduce: bf16 is not a reduction type");
  if (p == 0) return;
  const uint64_t sz = dtype_size(dt);
  if (bytes % (uint64_t(p) * sz))
    raise(MICS_TYPE_MISMATCH, "all_reduce: buffer of " + std::to_string(bytes) + " bytes is not divisible into " +
                                  std::to_string(p) + " chunks of whole " + std::to_string(sz) + "-byte elements");
  const uint64_t bs = round_up(bytes, kStage);
  const uint64_t b = s.block(bs * uint64_t(p));
  std::vector<void*> bp(static_cast<size_t>(p));
  for (int i = 0; i < p; ++i) {
    bp[size_t(i)] = s.at(b, ranks[i], uint64_t(i) * bs);
    s.h2d(ranks[i], bp[size_t(i)], bufs[i], bytes);
  }
  s.each([&](mics_ctx* m) { all_reduce(m, ranks, p, bp.data(), bytes / sz, dt); });
  for (int j = 0; j < p; ++j) s.d2h(ranks[j], out[j], bp[size_t(j)], bytes);
  s.finish();
}

void host_hier_all_gather(mics_ctx* ctx, int n, int p, int k, const void* const* shards, uint64_t chunk,
                          void* const* out, int corrupt) {
  if (n < 1 || n > ctx->n)
    raise(MICS_SHAPE_ERROR, "cluster has " + std::to_string(n) + " ranks but the context has " +
                                std::to_string(ctx->n));  // collectives.cpp:200-202
  Staging s(ctx);
  const uint64_t cs = round_up(chunk, kStage), os = round_up(uint64_t(p) * chunk, kStage);
  const uint64_t in = s.block(cs * uint64_t(n)), ob = s.block(os * uint64_t(n));
  std::vector<const void*> ip(static_cast<size_t>(n));
  std::vector<void*> op(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    ip[size_t(i)] = s.at(in, i, uint64_t(i) * cs);
    op[size_t(i)] = s.at(ob, i, uint64_t(i) * os);
    s.h2d(i, const_cast<void*>(ip[size_t(i)]), shards[i], chunk);
  }
  s.each([&](mics_ctx* m) { hier_all_gather(m, n, p, k, ip.data(), chunk, op.data(), corrupt); });
  for (int j = 0; j < n; ++j) s.d2h(j, out[j], op[size_t(j)], uint64_t(p) * chunk);
  s.finish();
}

void host_batched_all_gather(mics_ctx* ctx, int count, const int* sizes, const int* ranks, const uint64_t* chunks,
                             const void* const* shards, void* const* out) {
  Staging s(ctx);
  std::vector<mics_ag_desc> d(static_cast<size_t>(std::max(count, 0)));
  std::vector<std::vector<const void*>> ip(d.size());
  std::vector<std::vector<void*>> op(d.size());
  uint64_t ro = 0;
  for (int b = 0; b < count; ++b) {
    const int p = sizes[b];
    check_group(ctx, ranks + ro, p);
    const uint64_t c = chunks[b], cs = round_up(c, kStage), os = round_up(uint64_t(p) * c, kStage);
    const uint64_t in = s.block(cs * uint64_t(p)), ob = s.block(os * uint64_t(p));
    for (int i = 0; i < p; ++i) {
      const int r = ranks[ro + uint64_t(i)];
      ip[size_t(b)].push_back(s.at(in, r, uint64_t(i) * cs));
      op[size_t(b)].push_back(s.at(ob, r, uint64_t(i) * os));
      s.h2d(r, const_cast<void*>(ip[size_t(b)].back()), shards[ro + uint64_t(i)], c);
    }
    d[size_t(b)] = mics_ag_desc{ranks + ro, p, ip[size_t(b)].data(), c, op[size_t(b)].data()};
    ro += uint64_t(p);
  }
  s.each([&](mics_ctx* m) { batched_all_gather(m, d.data(), count); });
  ro = 0;
  for (int b = 0; b < count; ++b) {
    for (int j = 0; j < sizes[b]; ++j)
      s.d2h(ranks[ro + uint64_t(j)], out[ro + uint64_t(j)], op[size_t(b)][size_t(j)], uint64_t(sizes[b]) * chunks[b]);
    ro += uint64_t(sizes[b]);
  }
  s.finish();
}

void host_batched_reduce_scatter(mics_ctx* ctx, int count, const int* sizes, const int* ranks, const uint64_t* bytes,
                                 const void* const* bufs, mics_dtype dt, void* const* out) {
  Staging s(ctx);
  if (dt == MICS_BF16) raise(MICS_TYPE_MISMATCH, "reduce_scatter: bf16 is not a reduction type");
  const uint64_t sz = dtype_size(dt);
  std::vector<mics_rs_desc> d(static_cast<size_t>(std::max(count, 0)));
  std::vector<std::vector<const void*>> ip(d.size());
  std::vector<std::vector<void*>> op(d.size());
  uint64_t ro = 0;
  for (int b = 0; b < count; ++b) {
    const int p = sizes[b];
    check_group(ctx, ranks + ro, p);
    if (p > 0 && bytes[b] % (uint64_t(p) * sz))
      raise(MICS_TYPE_MISMATCH, "batched_reduce_scatter: buffer set " + std::to_string(b) +
                                    " is not divisible into whole chunks");
    const uint64_t bs = round_up(bytes[b], kStage), cb = p ? bytes[b] / uint64_t(p) : 0, cs = round_up(cb, kStage);
    const uint64_t in = s.block(bs * uint64_t(p)), ob = s.block(cs * uint64_t(p));
    for (int i = 0; i < p; ++i) {
      const int r = ranks[ro + uint64_t(i)];
      ip[size_t(b)].push_back(s.at(in, r, uint64_t(i) * bs));
      op[size_t(b)].push_back(s.at(ob, r, uint64_t(i) * cs));
      s.h2d(r, const_cast<void*>(ip[size_t(b)].back()), bufs[ro + uint64_t(i)], bytes[b]);
    }
    d[size_t(b)] = mics_rs_desc{ranks + ro, p, ip[size_t(b)].data(), bytes[b] / sz, bytes[b] / sz, op[size_t(b)].data()};
    ro += uint64_t(p);
  }
  s.each([&](mics_ctx* m) { batched_reduce_scatter(m, d.data(), count, dt, dt, 1.0, MICS_RS_STORE); });
  ro = 0;
  for (int b = 0; b < count; ++b) {
    const uint64_t cb = sizes[b] ? bytes[b] / uint64_t(sizes[b]) : 0;
    for (int j = 0; j < sizes[b]; ++j)
      s.d2h(ranks[ro + uint64_t(j)], out[ro + uint64_t(j)], op[size_t(b)][size_t(j)], cb);
    ro += uint64_t(sizes[b]);
  }
  s.finish();
}

}  // namespace mics
