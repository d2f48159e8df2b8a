// 2-hop gradient synchronisation (sync_schedule.hpp) on the device.
//
// mics_sync is SyncState<T> (sync_schedule.hpp:45-51) for every rank of the job,
// with the shard resident in the symmetric arena.  The schedule keeps the
// reference's state machine (check_micro_step :87-103 -> MICS_BOUNDARY_VIOLATION),
// its SyncEvent log (:27-32, byte counts of :142-144, :179-182, :219-222) and its
// traffic accounting; the data movement is the sm_100a pull engines:
//   micro-step  (:118-147) one k_reduce launch over every partition group and
//               segment: shard (+)= fold_{i<p} grad_i (ascending position)
//   boundary    (:153-185) k_reduce in place inside every replication group, then
//               k_copy (reference AR) or k_adam (AR's all-gather fused with Adam)
//   alternative (:189-232) AR over all n ranks into scratch + owned-chunk accumulate
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"
#include "sync.h"

namespace mics {

namespace {
void check_window(const mics_sync* st, bool at_boundary) {  // check_micro_step, sync_schedule.hpp:87-103
  if (at_boundary && st->micro_step != st->s)
    raise(MICS_BOUNDARY_VIOLATION, "boundary sync requires micro_step = s, have " + std::to_string(st->micro_step) +
                                       " of " + std::to_string(st->s));
  if (!at_boundary && st->micro_step >= st->s)
    raise(MICS_BOUNDARY_VIOLATION, "micro-step past accumulation boundary (micro_step = s = " +
                                       std::to_string(st->s) + ")");
}
std::vector<int> iota_ranks(int first, int count, int stride) {
  std::vector<int> r(static_cast<size_t>(count));
  for (int i = 0; i < count; ++i) r[size_t(i)] = first + i * stride;
  return r;
}
}  // namespace

mics_sync* sync_create(mics_ctx* ctx, int p, int s, int nseg, const uint64_t* seg_len, mics_dtype acc_t,
                       uint32_t align) {
  const int n = ctx->n;
  if (p < 1 || p > n)  // build_group_layout, topology.cpp:22-27
    raise(MICS_OUT_OF_RANGE, "partition size p=" + std::to_string(p) + " must satisfy 1 <= p <= n=" +
                                 std::to_string(n));
  if (n % p) raise(MICS_NON_DIVISIBLE, "partition size p=" + std::to_string(p) + " does not divide n=" +
                                           std::to_string(n));
  if (s < 1) raise(MICS_OUT_OF_RANGE, "micro-step count s must be >= 1");  // make_sync_states :61
  if (nseg < 1 || !seg_len) raise(MICS_OUT_OF_RANGE, "need at least one gradient segment");
  if (acc_t == MICS_BF16) raise(MICS_TYPE_MISMATCH, "shard accumulate type must be i64, f32 or f64");
  if (align < 1) align = 1;
  auto* st = new mics_sync();
  st->ctx = ctx;
  st->n = n;
  st->p = p;
  st->s = s;
  st->nseg = nseg;
  st->acc_t = acc_t;
  uint64_t so = 0, go = 0;
  for (int i = 0; i < nseg; ++i) {
    const uint64_t c = round_up(ceil_div(seg_len[i], uint64_t(p)), align);  // owned_chunk_elems :53-56
    st->len.push_back(seg_len[i]);
    st->chunk.push_back(c);
    st->shard_off.push_back(so);
    st->grad_off.push_back(go);
    so += c;
    go += c * uint64_t(p);
  }
  st->shard_elems = so;
  st->grad_elems = go;
  const int r = n / p;
  // boundary slices: position i of a replication group reduces slice i (16-byte aligned)
  st->sub = round_up(ceil_div(so, uint64_t(r)), 4);
  const uint64_t sz = dtype_size(acc_t);
  st->shard = alloc_sym(ctx, std::max<uint64_t>(uint64_t(r) * st->sub, 1) * sz);
  // SyncState shards start at T{} (make_sync_states :65)
  MICS_CUDA(cudaMemsetAsync(ctx->base + st->shard.offset, 0, st->shard.stride * uint64_t(ctx->per), ctx->stream));
  return st;
}

// ---- micro-step: one reduce launch over all partition groups and segments
Launch build_micro_launch(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale, int mode,
                          bool persistent, bool record, int entry, int exit, const mics_buf* shard_override,
                          int seg_lo, int seg_hi) {
  if (seg_hi < 0) seg_hi = st->nseg;  // segments [seg_lo, seg_hi) (a layer group of the step driver)
  mics_ctx* ctx = st->ctx;
  const int p = st->p;
  const mics_buf shard = shard_override ? *shard_override : st->shard;
  const uint64_t szg = dtype_size(grad_t), sza = dtype_size(st->acc_t);
  RedPlan plan(grad_t);
  uint64_t mask = 0;
  for (int g = 0; g < st->n / p; ++g) {
    const std::vector<int> ranks = iota_ranks(g * p, p, 1);
    if (record) {
      for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j)
          if (i != j)
            for (int q = seg_lo; q < seg_hi; ++q) ctx->record(g * p + i, g * p + j, st->chunk[size_t(q)] * szg);
    }
    mask |= ctx->peer_mask(ranks.data(), p);
    for (int j = 0; j < p; ++j) {
      const int rank = g * p + j;
      if (!ctx->local(rank)) continue;
      for (int q = seg_lo; q < seg_hi; ++q) {
        const uint64_t c = st->chunk[size_t(q)], first = uint64_t(j) * c;
        std::vector<const void*> srcs(static_cast<size_t>(p));
        for (int i = 0; i < p; ++i)
          srcs[size_t(i)] = ctx->rank_ptr(grads, g * p + i) + goff + (st->grad_off[size_t(q)] + first) * szg;
        const uint64_t len = st->len[size_t(q)];
        plan.add(srcs, ctx->rank_ptr(shard, rank) + st->shard_off[size_t(q)] * sza, c, len > first ? len - first : 0);
      }
    }
  }
  // later readers of the accumulated shards (the boundary's reduce-scatter) enter through
  // their own barrier: no publication needed
  return make_reduce_launch(ctx, plan, grad_t, st->acc_t, scale, mode, ctx->barrier(mask, entry, exit, 0, 0),
                            persistent);
}

void micro_step(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale, int mode) {
  check_window(st, false);
  if (!(grad_t == st->acc_t || (grad_t == MICS_BF16 && st->acc_t == MICS_F32)))
    raise(MICS_TYPE_MISMATCH, "gradient type does not match the shard type");
  if (goff + st->grad_elems * dtype_size(grad_t) > grads.stride)
    raise(MICS_SIZE_MISMATCH, "gradient buffer smaller than the padded gradient layout");
  Launch l = build_micro_launch(st, grads, goff, grad_t, scale, mode, false, true, 1, 1);
  enqueue(st->ctx, l);
  uint64_t cs = 0;
  for (uint64_t c : st->chunk) cs += c;
  for (int g = 0; g < st->n / st->p; ++g)  // :142-144
    st->events.push_back({st->micro_step, 0, g, int64_t(uint64_t(st->p - 1) * cs * dtype_size(grad_t))});
  st->micro_step++;
}

// ---- boundary
BoundaryLaunches build_boundary(mics_sync* st, const mics_adam* adam, bool persistent, bool record) {
  mics_ctx* ctx = st->ctx;
  const int n = st->n, p = st->p, r = n / p;
  const uint64_t sza = dtype_size(st->acc_t), sub = st->sub;
  BoundaryLaunches out;
  uint64_t rmask = 0, pmask = 0;
  for (int j = 0; j < p; ++j) {
    const std::vector<int> ranks = iota_ranks(j, r, p);
    rmask |= ctx->peer_mask(ranks.data(), r);
  }
  for (int g = 0; g < n / p; ++g) {
    const std::vector<int> ranks = iota_ranks(g * p, p, 1);
    pmask |= ctx->peer_mask(ranks.data(), p);
  }
  if (record && r > 1) {  // all_reduce over the padded shard: RS + AG messages (collectives.cpp:185-190)
    const uint64_t padded = ceil_div(st->shard_elems, uint64_t(r)) * uint64_t(r);
    for (int j = 0; j < p; ++j)
      for (int a = 0; a < r; ++a)
        for (int b = 0; b < r; ++b)
          if (a != b) {
            ctx->record(j + a * p, j + b * p, padded / uint64_t(r) * sza);
            ctx->record(j + a * p, j + b * p, padded / uint64_t(r) * sza);
          }
  }
  if (r > 1) {  // reduce-scatter in place: position i folds slice i of every replica's shard
    RedPlan rs(st->acc_t);
    for (int rho = 0; rho < n; ++rho) {
      if (!ctx->local(rho)) continue;
      const int j = rho % p, i = rho / p;
      std::vector<const void*> srcs(static_cast<size_t>(r));
      for (int q = 0; q < r; ++q) srcs[size_t(q)] = ctx->rank_ptr(st->shard, j + q * p) + uint64_t(i) * sub * sza;
      rs.add(srcs, ctx->rank_ptr(st->shard, rho) + uint64_t(i) * sub * sza, sub, sub);
    }
    out.rs = make_reduce_launch(ctx, rs, st->acc_t, st->acc_t, 1.0, MICS_RS_STORE, ctx->barrier(rmask, 1, 1),
                                persistent);
    out.has_rs = true;
  }
  if (adam) {
    if (st->acc_t != MICS_F32) raise(MICS_TYPE_MISMATCH, "the fused Adam update needs an f32 shard");
    AdamPlan ap;
    const uint64_t asub = r > 1 ? sub : round_up(std::max<uint64_t>(st->shard_elems, 1), 4);
    for (int rho = 0; rho < n; ++rho) {
      if (!ctx->local(rho)) continue;
      const int j = rho % p;
      std::vector<const void*> srcs(static_cast<size_t>(r));
      for (int q = 0; q < r; ++q) srcs[size_t(q)] = ctx->rank_ptr(st->shard, j + q * p);
      uint16_t* pb = adam->param_bf16.stride ? reinterpret_cast<uint16_t*>(ctx->rank_ptr(adam->param_bf16, rho)) : nullptr;
      ap.add(srcs, reinterpret_cast<float*>(ctx->rank_ptr(adam->param, rho)),
             reinterpret_cast<float*>(ctx->rank_ptr(adam->exp_avg, rho)),
             reinterpret_cast<float*>(ctx->rank_ptr(adam->exp_avg_sq, rho)), pb,
             adam->write_grad ? reinterpret_cast<float*>(ctx->rank_ptr(st->shard, rho)) : nullptr, st->shard_elems,
             asub);
    }
    // exit barrier with the replication group (done reading its slices) and the
    // partition group (their next all-gather reads the parameters updated here)
    out.ag = make_adam_launch(ctx, ap,
                              make_adam_scalars(adam->lr, adam->beta1, adam->beta2, adam->eps, adam->weight_decay,
                                                adam->step, adam->grad_scale),
                              ctx->barrier(rmask | pmask, 0, 1), persistent);
    out.has_ag = true;
  } else if (r > 1) {
    CopyPlan ag;
    for (int rho = 0; rho < n; ++rho) {
      if (!ctx->local(rho)) continue;
      const int j = rho % p, i = rho / p;
      std::vector<std::pair<const void*, std::vector<void*>>> items;
      for (int q = 0; q < r; ++q) {
        if (q == i) continue;
        const uint64_t o = uint64_t(q) * sub * sza;
        items.push_back({ctx->rank_ptr(st->shard, j + q * p) + o, {ctx->rank_ptr(st->shard, rho) + o}});
      }
      ag.add_group(items, sub * sza);
    }
    out.ag = make_copy_launch(ctx, ag, ctx->barrier(rmask, 0, 1), persistent);
    out.has_ag = true;
  }
  return out;
}

// The boundary restricted to shard elements [lo, hi) — one layer group of the step
// driver's pipelined boundary — on accumulator buffer `shard` and barrier channel
// `chan`.  Same fold order and Adam as build_boundary: the range is split into r
// slices of ceil(len/r) (rounded to 4) and position i reduces slice i in place.
BoundaryLaunches build_boundary_range(mics_sync* st, const mics_adam* adam, mics_buf shard, uint64_t lo, uint64_t hi,
                                      int chan, int rs_chan) {
  mics_ctx* ctx = st->ctx;
  const int n = st->n, p = st->p, r = n / p;
  const uint64_t len = hi - lo;
  const uint64_t subg = round_up(ceil_div(len, uint64_t(r)), 4);
  BoundaryLaunches out;
  uint64_t rmask = 0, pmask = 0;
  for (int j = 0; j < p; ++j) {
    const std::vector<int> ranks = iota_ranks(j, r, p);
    rmask |= ctx->peer_mask(ranks.data(), r);
  }
  for (int g = 0; g < n / p; ++g) {
    const std::vector<int> ranks = iota_ranks(g * p, p, 1);
    pmask |= ctx->peer_mask(ranks.data(), p);
  }
  if (r > 1) {
    RedPlan rs(MICS_F32);
    for (int rho = 0; rho < n; ++rho) {
      if (!ctx->local(rho)) continue;
      const int j = rho % p, i = rho / p;
      const uint64_t start = lo + uint64_t(i) * subg;
      const uint64_t elems = start < hi ? std::min(subg, hi - start) : 0;
      std::vector<const void*> srcs(static_cast<size_t>(r));
      for (int q = 0; q < r; ++q) srcs[size_t(q)] = ctx->rank_ptr(shard, j + q * p) + start * 4;
      rs.add(srcs, ctx->rank_ptr(shard, rho) + start * 4, elems, elems);
    }
    out.rs = make_reduce_launch(ctx, rs, MICS_F32, MICS_F32, 1.0, MICS_RS_STORE, ctx->barrier(rmask, 1, 1, rs_chan < 0 ? chan : rs_chan), true);
    out.has_rs = true;
  }
  AdamPlan ap;
  // Two local replicas of the same position need the same reduced gradient: one job
  // pulls it once and updates both (each from its own state).  MICS_ADAM_DEDUP=0 keeps
  // one job per rank.
  const char* de = std::getenv("MICS_ADAM_DEDUP");
  const bool dedup = !(de && de[0] == '0');
  std::vector<char> merged(static_cast<size_t>(n), 0);
  auto bf_of = [&](int rho) -> uint16_t* {
    return adam->param_bf16.stride ? reinterpret_cast<uint16_t*>(ctx->rank_ptr(adam->param_bf16, rho)) + lo : nullptr;
  };
  for (int rho = 0; rho < n; ++rho) {
    if (!ctx->local(rho) || merged[size_t(rho)]) continue;
    const int j = rho % p;
    std::vector<const void*> srcs(static_cast<size_t>(r));
    for (int q = 0; q < r; ++q) srcs[size_t(q)] = ctx->rank_ptr(shard, j + q * p) + lo * 4;
    ap.add(srcs, reinterpret_cast<float*>(ctx->rank_ptr(adam->param, rho)) + lo,
           reinterpret_cast<float*>(ctx->rank_ptr(adam->exp_avg, rho)) + lo,
           reinterpret_cast<float*>(ctx->rank_ptr(adam->exp_avg_sq, rho)) + lo, bf_of(rho), nullptr, len,
           r > 1 ? subg : round_up(std::max<uint64_t>(len, 1), 4));
    if (!dedup || len == 0) continue;
    for (int rho2 = rho + p; rho2 < n; rho2 += p)
      if (ctx->local(rho2) && !merged[size_t(rho2)]) {
        ap.add_replica(reinterpret_cast<float*>(ctx->rank_ptr(adam->param, rho2)) + lo,
                       reinterpret_cast<float*>(ctx->rank_ptr(adam->exp_avg, rho2)) + lo,
                       reinterpret_cast<float*>(ctx->rank_ptr(adam->exp_avg_sq, rho2)) + lo, bf_of(rho2));
        merged[size_t(rho2)] = 1;
        break;
      }
  }
  out.ag = make_adam_launch(ctx, ap,
                            make_adam_scalars(adam->lr, adam->beta1, adam->beta2, adam->eps, adam->weight_decay,
                                              adam->step, adam->grad_scale),
                            ctx->barrier(rmask | pmask, 0, 1, chan), true);
  out.has_ag = true;
  return out;
}

// K9: the boundary of shard range [lo, hi) (one layer group of the overlapped tail) as ONE
// launch: the replication-group reduce-scatter of every local rank's slice, published
// block by block into every replica's flags, then Adam pulling each block once its
// owner published it (FbRsJob / FbAdJob).  Same folds and Adam as build_boundary_range;
// slices are whole blocks (fb_block()).  `flags`: per rank [groups][r][nblk] u64; `g`: this
// group's index.  Entry barrier with the replication group (every replica's last
// micro-step reduce-scatter of the group is done), exit barrier with the replication
// and partition groups (done reading the owners' slices; parameters published).
uint32_t fb_block() {
  static const uint32_t b = [] {
    const char* e = std::getenv("MICS_FB_BLOCK");
    const long v = e ? std::atol(e) : 16384;
    return uint32_t(std::max<long>(8192, round_up(uint64_t(std::max<long>(v, 1)), 8192)));
  }();
  return b;
}

Launch build_boundary_fused_range(mics_sync* st, const mics_adam* adam, uint64_t lo, uint64_t hi, mics_buf flags,
                                  int g, int G, uint32_t nblk_max, int chan) {
  mics_ctx* ctx = st->ctx;
  const int n = st->n, p = st->p, r = n / p;
  if (r > kTailMaxR) raise(MICS_SHAPE_ERROR, "fused boundary: more than 8 replicas");
  const uint32_t blk = fb_block();
  const uint64_t len = hi - lo, sub = round_up(ceil_div(len, uint64_t(r)), blk);
  const uint32_t nblk = uint32_t(sub / blk);
  if (nblk > nblk_max) raise(MICS_CONFIG_ERROR, "fused boundary: flag array too small");
  uint64_t rmask = 0, pmask = 0;
  for (int j = 0; j < p; ++j) {
    const std::vector<int> ranks = iota_ranks(j, r, p);
    rmask |= ctx->peer_mask(ranks.data(), r);
  }
  for (int gg = 0; gg < n / p; ++gg) {
    const std::vector<int> ranks = iota_ranks(gg * p, p, 1);
    pmask |= ctx->peer_mask(ranks.data(), p);
  }
  auto shard = [&](int rank) { return reinterpret_cast<float*>(ctx->rank_ptr(st->shard, rank)) + lo; };
  auto flag_of = [&](int rank, int pos) {  // rank's flags for owner `pos` in group g
    return reinterpret_cast<uint64_t*>(ctx->rank_ptr(flags, rank)) + (uint64_t(g) * r + pos) * nblk_max;
  };
  const uint64_t ticket_off = uint64_t(G) * r * nblk_max + g;  // after every group's flags
  std::vector<FbRsJob> rs;
  std::vector<FbAdJob> ad;
  bool sys = false;
  Launch l;
  l.kind = Launch::FBND;
  for (int rho = 0; rho < n; ++rho) {
    if (!ctx->local(rho)) continue;
    if (!l.fb.ticket)  // the first local rank's copy
      l.fb.ticket = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(ctx->rank_ptr(flags, rho)) + ticket_off);
    const int j = rho % p, i = rho / p;
    for (int q = 0; q < r; ++q) sys |= !ctx->local(j + q * p);
    const uint64_t start = uint64_t(i) * sub, elems = start < len ? std::min(sub, len - start) : 0;
    if (elems) {
      FbRsJob J;
      std::memset(&J, 0, sizeof(J));
      for (int q = 0; q < r; ++q) {
        J.src[q] = shard(j + q * p) + start;
        J.flag[q] = flag_of(j + q * p, i);
        (ctx->local(j + q * p) ? l.hbm_bytes : l.remote_bytes) += elems * 4;
      }
      J.own = shard(rho) + start;
      J.elems = elems;
      J.r = uint32_t(r);
      l.hbm_bytes += elems * 4;
      rs.push_back(J);
    }
  }
  // Adam: one job per local rank; a second local replica of the same position shares it
  std::vector<char> merged(static_cast<size_t>(n), 0);
  auto bf_of = [&](int rho) -> uint16_t* {
    return adam->param_bf16.stride ? reinterpret_cast<uint16_t*>(ctx->rank_ptr(adam->param_bf16, rho)) + lo : nullptr;
  };
  auto f32 = [&](mics_buf b, int rho) { return reinterpret_cast<float*>(ctx->rank_ptr(b, rho)) + lo; };
  for (int rho = 0; rho < n; ++rho) {
    if (!ctx->local(rho) || merged[size_t(rho)] || len == 0) continue;
    const int j = rho % p;
    FbAdJob J;
    std::memset(&J, 0, sizeof(J));
    for (int q = 0; q < r; ++q) {
      J.owner[q] = shard(j + q * p);
      const uint64_t a = std::min<uint64_t>(uint64_t(q) * sub, len), b = std::min<uint64_t>((uint64_t(q) + 1) * sub, len);
      (ctx->local(j + q * p) ? l.hbm_bytes : l.remote_bytes) += (b - a) * 4;
    }
    J.flags = flag_of(rho, 0);
    J.prm = f32(adam->param, rho);
    J.m = f32(adam->exp_avg, rho);
    J.v = f32(adam->exp_avg_sq, rho);
    J.bf = bf_of(rho);
    l.hbm_bytes += len * (24 + (J.bf ? 2 : 0));
    for (int rho2 = rho + p; rho2 < n; rho2 += p)
      if (ctx->local(rho2) && !merged[size_t(rho2)]) {
        J.prm2 = f32(adam->param, rho2);
        J.m2 = f32(adam->exp_avg, rho2);
        J.v2 = f32(adam->exp_avg_sq, rho2);
        J.bf2 = bf_of(rho2);
        l.hbm_bytes += len * (24 + (J.bf2 ? 2 : 0));
        merged[size_t(rho2)] = 1;
        break;
      }
    J.elems = len;
    J.sub = sub;
    J.fstride = nblk_max;
    ad.push_back(J);
  }
  l.fb.nrs = int(rs.size());
  l.fb.nad = int(ad.size());
  l.fb.r = uint32_t(r);
  l.fb.nblk = nblk;
  l.fb.blk = blk;
  l.ndesc = int(rs.size() + ad.size());
  // grid: one resident wave (measured: 1 CTA per SM 4.55 ms, one CTA per item 3.26 ms,
  // the wave of 2 per SM 3.18 ms; C3 N=4 boundary)
  const uint64_t wave = uint64_t(ctx->nsm) * uint64_t(ctx->occ_fbnd);
  // lag: Adam items of block t are taken two waves of CTAs after the fold of block t
  // (MICS_FB_LAG overrides), so they rarely wait (C3, 4 GPUs: 1 wave 3.29 ms, 2 waves
  // 3.18 ms, 8 rounds 3.64 ms)
  const uint32_t per_round = uint32_t(rs.size() + ad.size() * size_t(r));
  const char* le = std::getenv("MICS_FB_LAG");
  l.fb.lag = le ? uint32_t(std::max(0, std::atoi(le))) : uint32_t(ceil_div(2 * wave, std::max<uint32_t>(per_round, 1))) + 1;
  // rounds t = 0 .. nblk + lag - 1: the fold of block t, then Adam of block t - lag
  l.ntiles = l.ndesc ? (nblk + l.fb.lag) * per_round : 0;
  l.grid = int(std::max<uint64_t>(std::min<uint64_t>(l.ntiles, wave), 1));
  l.hier_sys = sys ? 1 : 0;
  l.adam = make_adam_scalars(adam->lr, adam->beta1, adam->beta2, adam->eps, adam->weight_decay, adam->step,
                             adam->grad_scale);
  l.bar = ctx->barrier(rmask | pmask, 1, 1, chan);
  if (l.ndesc) {  // one blob: fold jobs, then Adam jobs
    const uint64_t o1 = round_up(sizeof(FbRsJob) * rs.size(), 16), bytes = o1 + sizeof(FbAdJob) * ad.size();
    MICS_CUDA(cudaMalloc(&l.d_desc, bytes));
    std::vector<char> blob(bytes, 0);
    if (!rs.empty()) std::memcpy(blob.data(), rs.data(), sizeof(FbRsJob) * rs.size());
    if (!ad.empty()) std::memcpy(blob.data() + o1, ad.data(), sizeof(FbAdJob) * ad.size());
    MICS_CUDA(cudaMemcpy(l.d_desc, blob.data(), bytes, cudaMemcpyHostToDevice));
    l.fb.rs = static_cast<const FbRsJob*>(l.d_desc);
    l.fb.ad = reinterpret_cast<const FbAdJob*>(static_cast<const char*>(l.d_desc) + o1);
  }
  return l;
}

void boundary(mics_sync* st, const mics_adam* adam) {
  check_window(st, true);
  BoundaryLaunches b = build_boundary(st, adam, false, true);
  if (b.has_rs) enqueue(st->ctx, b.rs);
  if (b.has_ag) enqueue(st->ctx, b.ag);
  const int r = st->n / st->p;
  const uint64_t padded = ceil_div(st->shard_elems, uint64_t(r)) * uint64_t(r);
  for (int j = 0; j < st->p; ++j)  // :179-182
    st->events.push_back(
        {st->s, 1, j, int64_t(2 * uint64_t(r - 1) * (padded / uint64_t(r)) * dtype_size(st->acc_t))});
  st->micro_step = 0;  // :184
}

// ---- alternative (DeepSpeed-default) schedule: all-reduce over all n ranks
// RS over all n ranks into the scratch buffer, AG of the reduced slices, then
// the owned chunk is accumulated into the shard (sync_schedule.hpp:189-224).
std::vector<Launch> build_alt(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale,
                              bool persistent, int acc_mode) {
  mics_ctx* ctx = st->ctx;
  const int n = st->n, p = st->p;
  const uint64_t szg = dtype_size(grad_t), sza = dtype_size(st->acc_t);
  if (!st->alt_ready) {  // per segment: n slices of ceil(p*chunk/n) elements (SPMD: same on every process)
    uint64_t off = 0;
    for (int q = 0; q < st->nseg; ++q) {
      const uint64_t sub = ceil_div(uint64_t(p) * st->chunk[size_t(q)], uint64_t(n));
      st->alt_sub.push_back(sub);
      st->alt_off.push_back(off);
      off += sub * uint64_t(n);
    }
    st->alt = alloc_sym(ctx, std::max<uint64_t>(off, 1) * sza);
    st->alt_ready = true;
  }
  std::vector<int> all = iota_ranks(0, n, 1);
  const uint64_t mask = ctx->peer_mask(all.data(), n);
  RedPlan rs(grad_t);
  CopyPlan ag;
  RedPlan acc(st->acc_t);
  for (int rho = 0; rho < n; ++rho) {
    if (!ctx->local(rho)) continue;
    for (int q = 0; q < st->nseg; ++q) {
      const uint64_t total = uint64_t(p) * st->chunk[size_t(q)], sub = st->alt_sub[size_t(q)];
      const uint64_t first = uint64_t(rho) * sub;
      const uint64_t elems = first < total ? std::min(sub, total - first) : 0;
      std::vector<const void*> srcs(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i)
        srcs[size_t(i)] = ctx->rank_ptr(grads, i) + goff + (st->grad_off[size_t(q)] + first) * szg;
      const uint64_t len = st->len[size_t(q)];
      rs.add(srcs, ctx->rank_ptr(st->alt, rho) + (st->alt_off[size_t(q)] + first) * sza, elems,
             len > first ? len - first : 0);
      std::vector<std::pair<const void*, std::vector<void*>>> items;
      uint64_t e2 = 0;
      for (int i = 0; i < n; ++i) {
        if (i == rho) continue;
        const uint64_t f2 = uint64_t(i) * sub;
        const uint64_t ei = f2 < total ? std::min(sub, total - f2) : 0;
        const uint64_t o = (st->alt_off[size_t(q)] + f2) * sza;
        if (ei == sub) items.push_back({ctx->rank_ptr(st->alt, i) + o, {ctx->rank_ptr(st->alt, rho) + o}});
        else ag.add(ctx->rank_ptr(st->alt, i) + o, {ctx->rank_ptr(st->alt, rho) + o}, ei * sza);  // ragged last slice
        e2 = sub;
      }
      ag.add_group(items, e2 * sza);
      const uint64_t c = st->chunk[size_t(q)];
      acc.add({ctx->rank_ptr(st->alt, rho) + (st->alt_off[size_t(q)] + uint64_t(rho % p) * c) * sza},
              ctx->rank_ptr(st->shard, rho) + st->shard_off[size_t(q)] * sza, c, c);
    }
  }
  std::vector<Launch> out;
  out.push_back(make_reduce_launch(ctx, rs, grad_t, st->acc_t, scale, MICS_RS_STORE, ctx->barrier(mask, 1, 1),
                                   persistent));
  out.push_back(make_copy_launch(ctx, ag, ctx->barrier(mask, 0, 1), persistent));
  out.push_back(make_reduce_launch(ctx, acc, st->acc_t, st->acc_t, 1.0, acc_mode, ctx->barrier(0, 0, 0),
                                   persistent));
  return out;
}

void alt_step(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale) {
  check_window(st, false);
  if (!(grad_t == st->acc_t || (grad_t == MICS_BF16 && st->acc_t == MICS_F32)))
    raise(MICS_TYPE_MISMATCH, "gradient type does not match the shard type");
  if (goff + st->grad_elems * dtype_size(grad_t) > grads.stride)
    raise(MICS_SIZE_MISMATCH, "gradient buffer smaller than the padded gradient layout");
  mics_ctx* ctx = st->ctx;
  const int n = st->n;
  const uint64_t szg = dtype_size(grad_t);
  for (const Launch& l : build_alt(st, grads, goff, grad_t, scale, false, MICS_RS_ACCUMULATE)) enqueue(ctx, l);
  const uint64_t padded = ceil_div(st->grad_elems, uint64_t(n)) * uint64_t(n);  // :200-201
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      if (a != b) {
        ctx->record(a, b, padded / uint64_t(n) * szg);
        ctx->record(a, b, padded / uint64_t(n) * szg);
      }
  st->events.push_back({st->micro_step, 2, 0, int64_t(2 * uint64_t(n - 1) * (padded / uint64_t(n)) * szg)});
  st->micro_step++;
}

void alt_boundary(mics_sync* st) {
  check_window(st, true);
  st->micro_step = 0;
}

}  // namespace mics
