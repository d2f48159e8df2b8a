// MiCS step driver: one global training step of the communication hot path,
// executed for real in the order the reference's simulator models it
// (simulator.cpp:265-280):
//   for each of s micro-steps:
//     forward pass  — per-layer parameter all-gather, layers 0..L-1
//     backward pass — per-layer parameter all-gather, layers L-1..0
//     micro-step sync — coalesced reduce-scatter of every layer's gradient inside
//                       the partition group (2-hop hop 1, sync_schedule.hpp:118-147)
//   boundary — replication-group all-reduce fused with sharded fp32 Adam (hop 2,
//              :153-185 + the optimizer the reference leaves out)
//
// Everything is planned once into device-resident descriptor tables (persistent
// Launches) and replayed every step.  Layout per rank (symmetric arena):
//   param_bf16 [shard]  master/m/v fp32 [shard]  gathered bf16 [2 or 3 x max layer]
//   grads [s x grad_elems] (resident) or [grad_elems] (generated each micro-step)
//   gradient accumulator = the mics_sync shard (fp32, padded to r*sub)
// Layer l's chunk is ceil(E_l/p) rounded up to 8 elements, so every all-gather
// and reduce-scatter descriptor is 16-byte aligned.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"
#include "sync.h"


namespace mics {

namespace {
constexpr uint32_t kAlignElems = 8;

void release(mics_step* st) {
  for (auto& v : st->ag)
    for (auto& l : v) l.release();
  for (auto& l : st->agm) l.release();
  for (auto& v : st->micro)
    for (auto& l : v) l.release();
  st->bnd.rs.release();
  st->bnd.ag.release();
  if (st->gexec) cudaGraphExecDestroy(st->gexec);
  for (auto& l : st->tail_rs) l.release();
  st->ftail.release();
  for (auto& b : st->tail_bnd) {
    b.rs.release();
    b.ag.release();
  }
  for (auto& l : st->tail_fb) l.release();
  for (auto e : st->ev_tail) cudaEventDestroy(e);
  for (auto e : st->ev_tail_rs) cudaEventDestroy(e);
  if (st->tail_rs_stream) cudaStreamDestroy(st->tail_rs_stream);

  if (st->ev_tail_done) cudaEventDestroy(st->ev_tail_done);
  for (auto e : st->ev_h2d) cudaEventDestroy(e);
  for (auto e : st->ev_rs_slot) cudaEventDestroy(e);
  if (st->ev_begin) cudaEventDestroy(st->ev_begin);
  for (cudaEvent_t e : {st->ev_g[0], st->ev_g[1], st->ev_free[0], st->ev_free[1], st->ev_fork, st->ev_jg, st->ev_jc})
    if (e) cudaEventDestroy(e);
  for (auto e : st->ev_wg) cudaEventDestroy(e);
  for (auto e : st->ev_rsd) cudaEventDestroy(e);
  for (auto e : st->ev_copied) cudaEventDestroy(e);
  for (auto& l : st->rs_local) l.release();
  if (st->gs) cudaStreamDestroy(st->gs);
  if (st->cs) cudaStreamDestroy(st->cs);
  if (st->copy_stream) cudaStreamDestroy(st->copy_stream);
  if (st->d_scalars) cudaFree(st->d_scalars);
}

// all-gather of layer l into gathered slot (l % gather_slots) of every local rank:
// flat (one k_copy stripe-group launch) or hierarchical (one k_hier launch; its epoch
// counter lives on barrier channel `chan`)
std::vector<Launch> build_layer_ag(mics_step* st, int l, int chan) {
  mics_ctx* ctx = st->ctx;
  mics_sync* sy = st->sync;
  const int p = sy->p, n = sy->n;
  const uint64_t c = sy->chunk[size_t(l)], cb = c * 2, soff = sy->shard_off[size_t(l)] * 2;
  const uint64_t goff = uint64_t(l % st->gather_slots) * st->gathered_half;
  auto G = [&](int r, uint64_t pos) { return ctx->rank_ptr(st->gathered, r) + goff + pos * cb; };
  std::vector<Launch> out;
  const int k = st->cfg.hier_k;
  if (k <= 0 || p <= k) {
    CopyPlan plan;
    for (int g = 0; g < n / p; ++g) {
      std::vector<std::pair<const void*, std::vector<void*>>> items;  // one stripe group per partition group
      for (int i = 0; i < p; ++i) {
        std::vector<void*> dsts;
        for (int j = 0; j < p; ++j)
          if (ctx->local(g * p + j)) dsts.push_back(G(g * p + j, uint64_t(i)));
        if (!dsts.empty()) items.emplace_back(ctx->rank_ptr(st->pbf16, g * p + i) + soff, std::move(dsts));
      }
      plan.add_group(items, cb);
    }
    // no barrier: shards are static between boundaries; the micro-step
    // reduce-scatter and Adam barriers order every write against these reads
    Launch l = make_copy_launch(ctx, plan, ctx->barrier(0, 0, 0), true);
    l.bar.dep_first = 0;  // independent of the previous layer's gather (PDL); see enqueue_gathers
    l.grid = ctx->grid_for(plan.tiles, ctx->occ_copy_indep);
    out.push_back(l);
    return out;
  }
  // hierarchical, one launch per layer visit: stage-1 tiles publish flags, stage-3 tiles
  // wait for them (kernels.cu k_hier).  No barrier: stage 1 reads the static shards; the
  // gather slots' write-after-read order follows from the flags (a rank completes visit
  // i+1 only after every node peer started it, i.e. finished visit i) and at most every
  // third visit reusing a slot — see k_hier and DESIGN §8 item 12.
  HierPlan plan = plan_hier(
      ctx, n, p, k, cb, 0, [&](int r) { return static_cast<const void*>(ctx->rank_ptr(st->pbf16, r) + soff); }, G,
      [&](int r) { return reinterpret_cast<uint64_t*>(ctx->rank_ptr(st->hflags, r)); }, st->hflag_tiles);
  out.push_back(make_hier_launch(ctx, plan, ctx->barrier(0, 0, 0), chan, true));
  return out;
}

// Hierarchical gathers of one micro-step in the comm-only step: 2L+1 k_hier launches for
// the V = 2L layer visits (forward 0..L-1, backward L-1..0); launch x runs stage 1 of
// visit x and stage 3 of visit x-1, so each visit's NVLink-bound stage 1 overlaps the
// previous visit's stage 3, with no barrier.  Launches are serial on each GPU; before
// its first stage-3 tile a CTA waits until every process hosting a node peer has
// completed launch x-1 (its done counter, published by that launch's last CTA) — the
// only cross-GPU wait, one-sided and one launch back.  Write-after-read: a rank's launch
// x starts after its launch x-1, which waited for the peers' launch x-2, so every
// peer read of a slot that launch x rewrites (visits x-3 and earlier, read in launches
// x-2 and earlier) is done; the turn's repeated layer rewrites identical bytes.
void build_hier_merged(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  mics_sync* sy = st->sync;
  const int L = st->cfg.nlayers, p = sy->p, n = sy->n, k = st->cfg.hier_k;
  std::vector<int> visits;
  for (int l = 0; l < L; ++l) visits.push_back(l);
  for (int l = L; l-- > 0;) visits.push_back(l);
  auto stage = [&](int v, int which) {
    const int l = visits[size_t(v)];
    const uint64_t cb = sy->chunk[size_t(l)] * 2, soff = sy->shard_off[size_t(l)] * 2;
    const uint64_t goff = uint64_t(l % st->gather_slots) * st->gathered_half;
    return plan_hier(
        ctx, n, p, k, cb, 0, [&](int r) { return static_cast<const void*>(ctx->rank_ptr(st->pbf16, r) + soff); },
        [&](int r, uint64_t pos) { return ctx->rank_ptr(st->gathered, r) + goff + pos * cb; },
        [&](int r) { return reinterpret_cast<uint64_t*>(ctx->rank_ptr(st->hflags, r)); }, st->hflag_tiles, which,
        which == 2 ? 1 : 0);
  };
  // processes hosting a node peer of a local rank (self excluded: its launch x-1 is done)
  uint64_t peers = 0;
  for (int r = 0; r < n; ++r) {
    if (!ctx->local(r)) continue;
    const int base = r / p * p, m = (r - base) / k;
    for (int j2 = 0; j2 < k; ++j2)
      if (ctx->process_of(base + m * k + j2) != ctx->wrank) peers |= 1ull << ctx->process_of(base + m * k + j2);
  }
  // G visits per launch (st->hier_group): launch y runs stage 1 of visits [yG, yG+G) and
  // stage 3 of visits [(y-1)G, yG); the slots (3G) keep the write-after-read argument
  // (a slot is rewritten at least three launches after the launch that wrote it)
  const int V = int(visits.size()), G = st->hier_group, Y = (V + G - 1) / G;
  auto group = [&](int y, int which) {
    HierPlan g;
    for (int v = y * G; v < std::min(V, (y + 1) * G); ++v) g = concat_hier(g, stage(v, which));
    return g;
  };
  for (int x = 0; x <= Y; ++x) {
    HierPlan plan;
    if (x < Y) plan = group(x, 1);
    const uint32_t n1 = plan.tiles;
    if (x > 0) plan = concat_hier(plan, group(x - 1, 2));
    Launch l = make_hier_launch(ctx, plan, ctx->barrier(0, 0, 0), 0, true);
    l.hier_merged = 1;
    l.hier_n1 = n1 < plan.tiles ? n1 : 0;  // both ranges present: interleave them
    l.hier_peers = ctx->ipc_ready ? peers : 0;
    st->agm.push_back(l);
  }
}

void enqueue_generate(mics_step* st, int t) {
  mics_ctx* ctx = st->ctx;
  const uint64_t szg = dtype_size(st->cfg.grad_t);
  const uint64_t off = uint64_t(t % st->gslots) * st->sync->grad_elems * szg;
  for (int r = 0; r < ctx->n; ++r) {
    if (!ctx->local(r)) continue;
    launch_generate(ctx->stream, ctx->rank_ptr(st->grads, r) + off, st->cfg.grad_t, st->cfg.seed, r, t, 0, 0,
                    st->sync->grad_elems, ctx->nsm * 8);
    ctx->launches++;
  }
}

bool generated(const mics_step* st) { return !st->cfg.resident_grads && !st->compute; }

// The boundary in order on the main stream: the replication-group reduce-scatter,
// then Adam fused with the all-reduce's all-gather phase.
void enqueue_boundary(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  st->adam_step++;
  const AdamScalars sc = make_adam_scalars(st->cfg.lr, st->cfg.beta1, st->cfg.beta2, st->cfg.eps,
                                           st->cfg.weight_decay, st->adam_step, st->adam.grad_scale);
  if (st->d_scalars && !st->capturing) {  // boundary kernels read the device copy once a graph exists
    DevScalars v{};
    v.sc = sc;
    launch_set_scalars(ctx->stream, st->d_scalars, v);
  }
  if (st->bnd.has_rs) enqueue(ctx, st->bnd.rs);
  if (st->bnd.has_ag) {
    st->bnd.ag.adam = sc;
    enqueue(ctx, st->bnd.ag);
  }
}

// Up to `groups` layer groups of about equal shard size, in forward order: layer l
// joins the group its shard midpoint falls in (empty groups vanish).
void plan_layer_groups(mics_step* st, int groups = 4) {
  if (!st->group_range.empty()) return;
  mics_sync* sy = st->sync;
  const int L = st->cfg.nlayers;
  // MICS_TAIL_GROUPS overrides the pipeline depth of the overlapped tail
  if (const char* e = std::getenv("MICS_TAIL_GROUPS")) groups = std::max(1, std::min(16, std::atoi(e)));
  const uint64_t G = uint64_t(std::min(groups, L)), S = sy->shard_elems;
  int prev = -1;
  for (int l = 0; l < L; ++l) {
    const uint64_t mid = sy->shard_off[size_t(l)] + sy->chunk[size_t(l)] / 2;
    const int g = int(std::min(G - 1, mid * G / std::max<uint64_t>(S, 1)));
    if (g != prev) {
      st->group_first_layer.push_back(l);
      st->group_range.push_back({sy->shard_off[size_t(l)], 0});
      prev = g;
    }
    st->group_range.back().second = sy->shard_off[size_t(l)] + sy->chunk[size_t(l)];
  }
}

// The overlapped tail: the last micro-step's reduce-scatter group by group on the main
// stream (channel 0); once group g is reduced, its boundary reduce-scatter + Adam run on
// the side stream (channel 1) while the main stream reduces group g+1.  Same fold order
// and Adam as the in-order boundary (build_boundary_range), so the bits are identical.
// clk (profile): everything in order on the main stream, events around each launch
// (even entries: reduce-scatter, odd: boundary).
void enqueue_tail(mics_step* st, std::vector<cudaEvent_t>* clk) {
  mics_ctx* ctx = st->ctx;
  const bool serial = clk != nullptr;
  cudaStream_t M = ctx->stream, S = serial ? M : ctx->side_stream;
  st->adam_step++;
  const AdamScalars sc = make_adam_scalars(st->cfg.lr, st->cfg.beta1, st->cfg.beta2, st->cfg.eps,
                                           st->cfg.weight_decay, st->adam_step, st->adam.grad_scale);
  if (!st->tail_fb.empty()) ++st->fb_epoch;  // this step's flag value of the fused boundaries
  if (st->d_scalars && !st->capturing) {
    DevScalars v{};
    v.sc = sc;
    v.epoch = st->fb_epoch;
    launch_set_scalars(M, st->d_scalars, v);
  }
  auto mark = [&]() {
    if (!clk) return;
    cudaEvent_t e;
    MICS_CUDA(cudaEventCreate(&e));
    MICS_CUDA(cudaEventRecord(e, M));
    clk->push_back(e);
  };
  // three streams: last RS per group (main, channel 0) -> boundary RS per group (its own
  // stream, channel 2: NVLink-bound) -> Adam per group (side stream, channel 1: HBM-bound),
  // so group g+1's boundary reduce-scatter runs under group g's Adam
  cudaStream_t R2 = serial ? M : st->tail_rs_stream;
  mark();
  if (!st->tail_fb.empty()) {  // K9: each group's boundary is one launch on its own stream (channel 2)
    for (size_t g = 0; g < st->tail_rs.size(); ++g) {
      enqueue(ctx, st->tail_rs[g], -1, M);
      mark();
      if (!serial) {
        MICS_CUDA(cudaEventRecord(st->ev_tail[g], M));
        MICS_CUDA(cudaStreamWaitEvent(R2, st->ev_tail[g], 0));
      }
      Launch& f = st->tail_fb[g];
      f.adam = sc;
      f.fb_epoch = st->fb_epoch;
      enqueue(ctx, f, -1, R2);
      mark();
    }
    if (!serial) {
      MICS_CUDA(cudaEventRecord(st->ev_tail_done, R2));
      MICS_CUDA(cudaStreamWaitEvent(M, st->ev_tail_done, 0));
    }
    return;
  }
  for (size_t g = 0; g < st->tail_rs.size(); ++g) {
    enqueue(ctx, st->tail_rs[g], -1, M);
    mark();
    if (!serial) {
      MICS_CUDA(cudaEventRecord(st->ev_tail[g], M));
      MICS_CUDA(cudaStreamWaitEvent(R2, st->ev_tail[g], 0));
    }
    BoundaryLaunches& b = st->tail_bnd[g];
    if (b.has_rs) enqueue(ctx, b.rs, -1, R2);
    if (!serial) {
      MICS_CUDA(cudaEventRecord(st->ev_tail_rs[g], R2));
      MICS_CUDA(cudaStreamWaitEvent(S, st->ev_tail_rs[g], 0));
    }
    b.ag.adam = sc;
    enqueue(ctx, b.ag, -1, S);
    mark();
  }
  if (!serial) {
    MICS_CUDA(cudaEventRecord(st->ev_tail_done, S));
    MICS_CUDA(cudaStreamWaitEvent(M, st->ev_tail_done, 0));
  }
}

// K8 plan: one job per (partition position j, layer) covering that layer's chunk of
// every replica of position j (all ranks are local: world == 1).
void build_fused_tail(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  mics_sync* sy = st->sync;
  const int n = sy->n, p = sy->p, r = n / p, L = st->cfg.nlayers, s = st->cfg.s;
  const uint64_t szg = dtype_size(st->cfg.grad_t);
  const uint64_t goff = uint64_t((s - 1) % st->gslots) * sy->grad_elems * szg;
  std::vector<TailJob> jobs;
  uint32_t tiles = 0;
  uint64_t bytes = 0;
  for (int j = 0; j < p; ++j)
    for (int l = 0; l < L; ++l) {
      TailJob J;
      std::memset(&J, 0, sizeof(J));
      const uint64_t c = sy->chunk[size_t(l)], so = sy->shard_off[size_t(l)], first = uint64_t(j) * c;
      const uint64_t len = sy->len[size_t(l)];
      for (int q = 0; q < r; ++q) {
        const int rho = q * p + j;  // replica q of position j (partition group q)
        J.acc[q] = reinterpret_cast<const float*>(ctx->rank_ptr(sy->shard, rho)) + so;
        for (int i = 0; i < p; ++i)
          J.grads[q * kTailMaxP + i] = reinterpret_cast<const uint8_t*>(
              ctx->rank_ptr(st->grads, q * p + i) + goff + (sy->grad_off[size_t(l)] + first) * szg);
        J.prm[q] = reinterpret_cast<float*>(ctx->rank_ptr(st->master, rho)) + so;
        J.m[q] = reinterpret_cast<float*>(ctx->rank_ptr(st->m, rho)) + so;
        J.v[q] = reinterpret_cast<float*>(ctx->rank_ptr(st->v, rho)) + so;
        J.bf[q] = reinterpret_cast<uint16_t*>(ctx->rank_ptr(st->pbf16, rho)) + so;
      }
      J.elems = c;
      J.valid = len > first ? len - first : 0;
      J.tile0 = tiles;
      tiles += uint32_t(ceil_div(c, kTailTile));
      jobs.push_back(J);
      // HBM per element: r x (acc + p gradients + p, m, v) read, r x (p, m, v, bf16) written
      bytes += c * uint64_t(r) * ((s > 1 ? 4 : 0) + uint64_t(p) * szg + 12 + 14);
    }
  Launch& t = st->ftail;
  t.kind = Launch::TAIL;
  t.in_t = st->cfg.grad_t;
  t.tail_r = r;
  t.tail_p = p;
  t.mode = s == 1 ? 1 : 0;  // zero-accumulate when the last micro-step is the first
  t.ndesc = int(jobs.size());
  t.ntiles = tiles;
  t.grid = ctx->grid_for(tiles, 2);
  t.bar = ctx->barrier(0, 0, 0);
  t.hbm_bytes = bytes;
  MICS_CUDA(cudaMalloc(&t.d_desc, jobs.size() * sizeof(TailJob)));
  MICS_CUDA(cudaMemcpy(t.d_desc, jobs.data(), jobs.size() * sizeof(TailJob), cudaMemcpyHostToDevice));
  st->fused_tail = true;
}

void enqueue_fused_tail(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  st->adam_step++;
  const AdamScalars sc = make_adam_scalars(st->cfg.lr, st->cfg.beta1, st->cfg.beta2, st->cfg.eps,
                                           st->cfg.weight_decay, st->adam_step, st->adam.grad_scale);
  if (st->d_scalars && !st->capturing) {
    DevScalars v{};
    v.sc = sc;
    launch_set_scalars(ctx->stream, st->d_scalars, v);
  }
  st->ftail.adam = sc;
  enqueue(ctx, st->ftail);
}

// forward then backward per-layer gathers.  The first gather of a step follows the
// boundary's Adam (which rewrote the shards it reads), so it waits for its
// predecessor; the others only depend on static shards.
// In-flight bound: every (slots-1)-th gather is a fence (dep_first 0), so at most
// `slots` consecutive gathers run at once.  Two gathers within `slots` positions
// of each other either hit different slots (layers a != b mod slots) or carry the
// same bytes (the same layer at the forward/backward turn): no write-after-write
// race on a slot.  step_create rejects empty layers, so every gather launches and
// the fence positions are the ones counted here.
void enqueue_gathers(mics_step* st, int t) {
  mics_ctx* ctx = st->ctx;
  if (!st->agm.empty()) {  // merged hierarchical sequence (k_hier orders itself: flags, serial launches)
    for (const Launch& x : st->agm) enqueue(ctx, x);
    return;
  }
  bool first = true;
  const int m = st->gather_slots - 1;
  int pos = 0;
  // only the flat gathers are independent; hierarchical launches keep their plan
  auto go = [&](const Launch& x) {
    int d = -1;
    if (x.bar.dep_first == 0 && !x.bar.mask) d = pos++ % m == m - 1 ? 0 : 2;
    if (first && t == 0) d = 1;
    first = false;
    enqueue(ctx, x, d);
  };
  for (size_t l = 0; l < st->layers.size(); ++l)
    for (auto& x : st->ag[l]) go(x);
  for (size_t l = st->layers.size(); l-- > 0;)
    for (auto& x : st->ag[l]) go(x);
}

void enqueue_sync(mics_step* st, int t) {
  for (auto& x : st->micro[size_t(t)]) enqueue(st->ctx, x);
}

void enqueue_micro(mics_step* st, int t) {
  enqueue_gathers(st, t);
  enqueue_sync(st, t);
}

// ---------------------------------------------------------------- step with compute
// Layer l = W_l [rows_l, h] (its gathered bf16 parameters); per rank and micro-step t:
//   forward   Y_l  = X_t · W_lᵀ                 (bf16, stored or recomputed)
//   backward  dX  += Y_l · W_l                  (fp32; the input gradient of the branch sum)
//             dW_l = Y_lᵀ · X_t -> grads slot    (the layer's gradient, f32/bf16)
// i.e. the exact gradients of 1/2 sum_l ||X W_lᵀ||^2.  Plans are built once.
void setup_compute(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  mics_sync* sy = st->sync;
  const mics_step_cfg& cfg = st->cfg;
  const int L = cfg.nlayers, s = cfg.s;
  st->T = cfg.tokens;
  st->h = cfg.hidden;
  st->recompute = cfg.recompute != 0;
  uint64_t ytot = 0, ymax = 0;
  for (int l = 0; l < L; ++l) {
    const uint64_t E = st->layers[size_t(l)];
    if (E % st->h) raise(MICS_SHAPE_ERROR, "step with compute: layer " + std::to_string(l) + " has " +
                                                std::to_string(E) + " parameters, not a multiple of hidden " +
                                                std::to_string(st->h));
    const uint64_t rows = E / st->h;
    st->rows.push_back(rows);
    st->ldy.push_back(round_up(rows, 8));
    st->yoff.push_back(st->recompute ? 0 : ytot);
    ytot += st->T * round_up(rows, 8);
    ymax = std::max(ymax, st->T * round_up(rows, 8));
  }
  const uint64_t xe = st->T * st->h;
  st->x = alloc_sym(ctx, uint64_t(s) * xe * 2);
  st->y = alloc_sym(ctx, (st->recompute ? ymax : ytot) * 2);
  st->dx = alloc_sym(ctx, xe * 4);
  const uint64_t szg = dtype_size(cfg.grad_t);
  for (int r = 0; r < ctx->n; ++r) {  // inputs of every micro-step (the "batch"), generated once
    if (!ctx->local(r)) continue;
    for (int t = 0; t < s; ++t)
      launch_generate(ctx->stream, ctx->rank_ptr(st->x, r) + uint64_t(t) * xe * 2, MICS_BF16, cfg.seed ^ 0xA11CEull,
                      r, t, 254, 0, xe, ctx->nsm * 8);
  }
  // Overlap resources (measured on 2 B200, C3, one rank per GPU, profiles/r1/compute/):
  //  - flat per-layer gathers run on the copy engines (cudaMemcpyAsync of each
  //    chunk, local or NVLink peer): no SM time, so the co-resident GEMM keeps its
  //    speed (k_copy under a GEMM slowed it ~20%); MICS_CE_GATHER=0 uses k_copy;
  //  - the reduce-scatters that run under the next micro-step's GEMMs get comm_sms
  //    CTAs and the GEMMs the other SMs (MICS_COMM_SMS, default 16; 0 = share every
  //    SM).  37.0 ms/step (k_copy, shared) -> 36.2 (copy engines) -> 35.0 (+16 SMs).
  st->comm_sms = 16;
  if (const char* e = std::getenv("MICS_COMM_SMS")) st->comm_sms = std::max(0, std::min(ctx->nsm - 2, std::atoi(e)));
  {
    const char* e = std::getenv("MICS_RS_OVERLAP");
    st->rs_overlap = !(e && e[0] == '0');
    if (!st->rs_overlap) st->comm_sms = 0;  // nothing runs beside the GEMMs but copy-engine gathers
  }
  {
    // partition groups that span processes: the reduce-scatter pulls over NVLink, so
    // stage it through the copy engines instead (see mics_step::ce_rs)
    bool remote_peers = false;
    for (int r = 0; r < ctx->n; ++r)
      if (ctx->local(r))
        for (int i = 0; i < cfg.p; ++i) remote_peers |= !ctx->local(r / cfg.p * cfg.p + i);
    const char* e = std::getenv("MICS_CE_RS");
    st->ce_rs = remote_peers && cfg.s > 1 && !(e && e[0] == '0');
    if (st->ce_rs) st->comm_sms = 0;  // only a short local fold runs beside the GEMMs
  }
  const int gemm_sms = st->comm_sms ? ctx->nsm - st->comm_sms : 0;
  const int T = int(st->T), h = int(st->h);
  for (int t = 0; t < s; ++t)
    for (int l = 0; l < L; ++l)
      for (int r = 0; r < ctx->n; ++r) {
        if (!ctx->local(r)) continue;
        const int rows = int(st->rows[size_t(l)]);
        const uint64_t ldy = st->ldy[size_t(l)];
        char* W = ctx->rank_ptr(st->gathered, r) + uint64_t(l % st->gather_slots) * st->gathered_half;
        char* X = ctx->rank_ptr(st->x, r) + uint64_t(t) * xe * 2;
        char* Y = ctx->rank_ptr(st->y, r) + st->yoff[size_t(l)] * 2;
        char* dX = ctx->rank_ptr(st->dx, r);
        char* dW = ctx->rank_ptr(st->grads, r) + (uint64_t(t % st->gslots) * sy->grad_elems + sy->grad_off[size_t(l)]) * szg;
        st->gfwd.push_back(plan_gemm(X, st->h, 0, W, st->h, 0, Y, ldy, MICS_BF16, T, rows, h, 0, gemm_sms));
        st->gdgrad.push_back(
            plan_gemm(Y, ldy, 0, W, st->h, 1, dX, st->h, MICS_F32, T, h, rows, l != L - 1, gemm_sms));
        st->gwgrad.push_back(plan_gemm(Y, ldy, 1, X, st->h, 1, dW, st->h, cfg.grad_t, rows, h, T, 0, gemm_sms));
      }
  // Gathers are on the critical path (layer l+1's GEMMs wait for them): highest
  // priority; GEMMs lowest, so a freed SM slot goes to a waiting gather first.
  int prio_lo = 0, prio_hi = 0;
  MICS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  MICS_CUDA(cudaStreamCreateWithPriority(&st->gs, cudaStreamNonBlocking, prio_hi));
  MICS_CUDA(cudaStreamCreateWithPriority(&st->cs, cudaStreamNonBlocking, prio_lo));
  // Overlapped collectives: comm_sms CTAs (or, when sharing every SM, one CTA per SM,
  // whose registers and shared-memory table fit beside a GEMM CTA).  The serialised
  // profile step keeps the full grids.
  {
    const char* e = std::getenv("MICS_CE_GATHER");
    st->ce_gather = !(e && e[0] == '0') && (cfg.hier_k <= 0 || cfg.p <= cfg.hier_k);
  }
  if (st->ce_gather) {
    for (int l = 0; l < L; ++l) {
      const uint64_t c = sy->chunk[size_t(l)], cb = c * 2, soff = sy->shard_off[size_t(l)] * 2;
      std::vector<mics_step::CeCopy> v;
      for (int r = 0; r < ctx->n; ++r) {
        if (!ctx->local(r)) continue;
        const int g = r / cfg.p;
        char* G = ctx->rank_ptr(st->gathered, r) + uint64_t(l % st->gather_slots) * st->gathered_half;
        for (int i = 0; i < cfg.p; ++i) v.push_back({G + uint64_t(i) * cb, ctx->rank_ptr(st->pbf16, g * cfg.p + i) + soff, cb});
      }
      st->ce.push_back(std::move(v));
    }
  }
  if (st->ce_rs) {
    const int p = cfg.p;
    uint64_t csum = 0;
    std::vector<uint64_t> cum;
    for (uint64_t c : sy->chunk) {
      cum.push_back(csum);
      csum += c;
    }
    st->stage = alloc_sym(ctx, uint64_t(p) * csum * szg);
    auto stage_ptr = [&](int r, int i, int q) {
      return ctx->rank_ptr(st->stage, r) + (uint64_t(i) * csum + cum[size_t(q)]) * szg;
    };
    for (int slot = 0; slot < st->gslots; ++slot) {
      const uint64_t goff = uint64_t(slot) * sy->grad_elems * szg;
      std::vector<std::vector<mics_step::CeCopy>> per_layer(static_cast<size_t>(L));
      for (int r = 0; r < ctx->n; ++r) {
        if (!ctx->local(r)) continue;
        const int g = r / p, j = r % p;
        for (int i = 0; i < p; ++i) {
          if (ctx->local(g * p + i)) continue;
          for (int q = 0; q < L; ++q) {
            const uint64_t c = sy->chunk[size_t(q)];
            per_layer[size_t(q)].push_back(
                {stage_ptr(r, i, q),
                 ctx->rank_ptr(st->grads, g * p + i) + goff + (sy->grad_off[size_t(q)] + uint64_t(j) * c) * szg,
                 c * szg});
          }
        }
      }
      st->ce_rs_copies.push_back(std::move(per_layer));
    }
    const uint64_t sza = dtype_size(sy->acc_t);
    for (int t = 0; t < s; ++t) {
      const uint64_t goff = uint64_t(t % st->gslots) * sy->grad_elems * szg;
      RedPlan plan(cfg.grad_t);
      for (int r = 0; r < ctx->n; ++r) {
        if (!ctx->local(r)) continue;
        const int g = r / p, j = r % p;
        for (int q = 0; q < L; ++q) {
          const uint64_t c = sy->chunk[size_t(q)], first = uint64_t(j) * c, len = sy->len[size_t(q)];
          std::vector<const void*> srcs(static_cast<size_t>(p));
          for (int i = 0; i < p; ++i)  // ascending position, local or staged: the same fold as the pull RS
            srcs[size_t(i)] = ctx->local(g * p + i)
                                  ? static_cast<const void*>(ctx->rank_ptr(st->grads, g * p + i) + goff +
                                                             (sy->grad_off[size_t(q)] + first) * szg)
                                  : static_cast<const void*>(stage_ptr(r, i, q));
          plan.add(srcs, ctx->rank_ptr(sy->shard, r) + sy->shard_off[size_t(q)] * sza, c, len > first ? len - first : 0);
        }
      }
      st->rs_local.push_back(make_reduce_launch(ctx, plan, cfg.grad_t, sy->acc_t, 1.0,
                                                t == 0 ? MICS_RS_ZERO_ACCUM : MICS_RS_ACCUMULATE,
                                                ctx->barrier(0, 0, 0), true));
    }
    uint64_t pmask = 0;
    for (int g = 0; g < ctx->n / p; ++g) {
      std::vector<int> ranks(static_cast<size_t>(p));
      for (int i = 0; i < p; ++i) ranks[size_t(i)] = g * p + i;
      pmask |= ctx->peer_mask(ranks.data(), p);
    }
    st->rs_bar.kind = Launch::BARRIER;
    st->rs_bar.bar = ctx->barrier(pmask, 1, 0, 2);
    st->ev_copied.resize(size_t(st->gslots));
    for (auto& e : st->ev_copied) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int lean = st->comm_sms ? st->comm_sms : ctx->nsm;
  for (auto& v : st->ag)
    for (auto& x : v) {
      st->ag_grid_full.push_back(x.grid);
      x.grid = std::min(x.grid, lean);
    }
  for (auto& v : st->micro)
    for (auto& x : v) {
      st->micro_grid_full.push_back(x.grid);
      x.grid = std::min(x.grid, lean);
    }
  for (cudaEvent_t* e : {&st->ev_g[0], &st->ev_g[1], &st->ev_free[0], &st->ev_free[1], &st->ev_fork, &st->ev_jg,
                         &st->ev_jc})
    MICS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  st->ev_wg.resize(size_t(st->gslots));
  st->ev_rsd.resize(size_t(st->gslots));
  for (auto& e : st->ev_wg) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : st->ev_rsd) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// Phase timing of a serialised step (profile): events around every gather and GEMM group.
struct PhaseClock {
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;  // phase of the interval ending at ev[i]
  cudaStream_t s = nullptr;
  void mark(int k) {
    cudaEvent_t e;
    MICS_CUDA(cudaEventCreate(&e));
    MICS_CUDA(cudaEventRecord(e, s));
    ev.push_back(e);
    kind.push_back(k);
  }
};
enum { PH_AG = 0, PH_RS = 1, PH_BND = 2, PH_GEN = 3, PH_GEMM = 4 };

// One step with compute.  serial: everything on ctx->stream in order (profiling);
// otherwise gathers on st->gs, GEMMs on st->cs, reduce-scatters + boundary on
// ctx->stream:
//   gather(l) waits ev_free[l%2] (the GEMMs that read that buffer last), GEMMs(l)
//   wait ev_g[l%2]; RS(t) waits ev_wg[slot] (all dW of t); the first dW GEMM of t
//   waits ev_rsd[slot] (the RS that read that gradient slot last).
// MICS_TRACE=<file>: eager compute steps record timing events around every gather,
// GEMM group and reduce-scatter on their own streams and append a timeline
// (op, t, l, start_ms, end_ms) to <file> — the overlap evidence without nsys.
struct Trace {
  struct Op {
    std::string name;
    int t, l;
    cudaEvent_t a, b;
  };
  std::vector<Op> ops;
  cudaEvent_t origin = nullptr;
  void begin(cudaStream_t s, const char* name, int t, int l) {
    Op o{name, t, l, nullptr, nullptr};
    MICS_CUDA(cudaEventCreate(&o.a));
    MICS_CUDA(cudaEventCreate(&o.b));
    MICS_CUDA(cudaEventRecord(o.a, s));
    ops.push_back(o);
  }
  void end(cudaStream_t s) { MICS_CUDA(cudaEventRecord(ops.back().b, s)); }
};
Trace* trace_for(mics_step* st) {
  static const char* path = std::getenv("MICS_TRACE");
  if (!path || st->capturing) return nullptr;
  return new Trace();
}
void trace_flush(Trace* tr, mics_ctx* ctx) {
  if (!tr) return;
  static const char* path = std::getenv("MICS_TRACE");
  MICS_CUDA(cudaStreamSynchronize(ctx->stream));
  MICS_CUDA(cudaDeviceSynchronize());
  FILE* f = std::fopen((std::string(path) + "." + std::to_string(ctx->wrank)).c_str(), "a");
  if (f) std::fprintf(f, "%d,step,-1,-1,0,0\n", ctx->wrank);  // one block per step
  for (auto& o : tr->ops) {
    float a = 0, b = 0;
    MICS_CUDA(cudaEventElapsedTime(&a, tr->origin, o.a));
    MICS_CUDA(cudaEventElapsedTime(&b, tr->origin, o.b));
    if (f) std::fprintf(f, "%d,%s,%d,%d,%.4f,%.4f\n", ctx->wrank, o.name.c_str(), o.t, o.l, a, b);
    cudaEventDestroy(o.a);
    cudaEventDestroy(o.b);
  }
  if (f) std::fclose(f);
  cudaEventDestroy(tr->origin);
  delete tr;
}

void enqueue_compute_step(mics_step* st, PhaseClock* clk) {
  mics_ctx* ctx = st->ctx;
  const bool serial = clk != nullptr;
  Trace* tr = serial ? nullptr : trace_for(st);
  if (tr) {
    MICS_CUDA(cudaEventCreate(&tr->origin));
    MICS_CUDA(cudaEventRecord(tr->origin, ctx->stream));
  }
  cudaStream_t M = ctx->stream, G = serial ? M : st->gs, C = serial ? M : st->cs;
  const int L = st->cfg.nlayers, s = st->cfg.s, per = ctx->per;
  auto rec = [&](cudaEvent_t e, cudaStream_t on) {
    if (!serial) MICS_CUDA(cudaEventRecord(e, on));
  };
  auto wait = [&](cudaStream_t on, cudaEvent_t e) {
    if (!serial) MICS_CUDA(cudaStreamWaitEvent(on, e, 0));
  };
  auto gemms = [&](const std::vector<GemmLaunch>& v, size_t base) {
    for (int li = 0; li < per; ++li) {
      launch_gemm(C, v[base + size_t(li)]);
      ctx->launches++;
    }
  };
  int cur_t = 0;
  // the serialised (profile) step runs the collectives with their full grids
  auto ag_index = [&](int l) {
    size_t i = 0;
    for (int k = 0; k < l; ++k) i += st->ag[size_t(k)].size();
    return i;
  };
  auto gather = [&](int l) {
    wait(G, st->ev_free[l % 2]);
    if (tr) tr->begin(G, "gather", cur_t, l);
    if (st->ce_gather && !serial) {
      for (const auto& c : st->ce[size_t(l)])
        MICS_CUDA(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToDevice, G));
    } else {
      size_t gi = ag_index(l);
      for (auto& x : st->ag[size_t(l)]) {
        Launch y = x;
        if (serial) y.grid = st->ag_grid_full[gi];
        ++gi;
        enqueue(ctx, y, -1, G);
      }
    }
    if (tr) tr->end(G);
    if (clk) clk->mark(PH_AG);
    rec(st->ev_g[l % 2], G);
    wait(C, st->ev_g[l % 2]);
  };
  // gathers and GEMMs wait for everything before this step on the main stream (the
  // previous boundary rewrote the parameter shards)
  rec(st->ev_fork, M);
  wait(G, st->ev_fork);
  wait(C, st->ev_fork);
  if (clk) clk->mark(-1);
  int pending = -1;  // micro-step whose copy-engine-staged reduce-scatter is still to do
  for (int t = 0; t < s; ++t) {
    const int slot = t % st->gslots;
    cur_t = t;
    for (int l = 0; l < L; ++l) {
      gather(l);
      if (tr) tr->begin(C, "fwd", t, l);
      gemms(st->gfwd, size_t(t * L + l) * size_t(per));
      if (tr) tr->end(C);
      if (clk) clk->mark(PH_GEMM);
      rec(st->ev_free[l % 2], C);
    }
    if (t >= st->gslots) wait(C, st->ev_rsd[size_t(slot)]);
    // the copy-engine-staged reduce-scatter of the previous micro-step rides on this
    // backward pass (gather stream, one layer's chunks after each layer's gather)
    const bool carry = st->ce_rs && !serial && pending >= 0;
    const int ps = carry ? pending % st->gslots : 0;
    if (carry) {
      MICS_CUDA(cudaStreamWaitEvent(G, st->ev_wg[size_t(ps)], 0));
      if (pending > 0)  // one staging buffer: the fold of micro-step pending-1 has read it
        MICS_CUDA(cudaStreamWaitEvent(G, st->ev_rsd[size_t((pending - 1) % st->gslots)], 0));
      enqueue(ctx, st->rs_bar, -1, G);  // peers' micro-step gradients are complete
    }
    for (int l = L; l-- > 0;) {
      gather(l);
      if (carry) {
        if (tr) tr->begin(G, "rs_copy", pending, l);
        for (const auto& c : st->ce_rs_copies[size_t(ps)][size_t(l)])
          MICS_CUDA(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToDevice, G));
        if (tr) tr->end(G);
      }
      const size_t base = size_t(t * L + l) * size_t(per);
      if (tr) tr->begin(C, "bwd", t, l);
      if (st->recompute) gemms(st->gfwd, base);
      gemms(st->gdgrad, base);
      gemms(st->gwgrad, base);
      if (tr) tr->end(C);
      if (clk) clk->mark(PH_GEMM);
      rec(st->ev_free[l % 2], C);
    }
    if (carry) {
      enqueue(ctx, st->rs_bar, -1, G);  // finished reading the peers' gradients
      MICS_CUDA(cudaEventRecord(st->ev_copied[size_t(ps)], G));
      MICS_CUDA(cudaStreamWaitEvent(M, st->ev_copied[size_t(ps)], 0));
      if (tr) tr->begin(M, "rs", pending, -1);
      enqueue(ctx, st->rs_local[size_t(pending)], -1, M);
      if (tr) tr->end(M);
      rec(st->ev_rsd[size_t(ps)], M);
      pending = -1;
    }
    rec(st->ev_wg[size_t(slot)], C);
    if (st->ce_rs && !serial && t != s - 1) {
      pending = t;  // carried by the next micro-step's backward pass
      continue;
    }
    wait(M, st->ev_wg[size_t(slot)]);
    if (tr) tr->begin(M, "rs", t, -1);
    const bool rs_under_compute = st->rs_overlap && t != s - 1;
    size_t mi = 0;
    for (int k = 0; k < t; ++k) mi += st->micro[size_t(k)].size();
    for (auto& x : st->micro[size_t(t)]) {
      Launch y = x;
      // the last micro-step's reduce-scatter overlaps no compute: full grid
      if (serial || !rs_under_compute) y.grid = st->micro_grid_full[mi];
      ++mi;
      enqueue(ctx, y, -1, M);
    }
    if (tr) tr->end(M);
    if (clk) clk->mark(PH_RS);
    rec(st->ev_rsd[size_t(slot)], M);
    if (!st->rs_overlap) wait(C, st->ev_rsd[size_t(slot)]);  // next micro-step's GEMMs after the RS
  }
  if (tr) tr->begin(M, "boundary", s, -1);
  enqueue_boundary(st);
  if (tr) tr->end(M);
  if (clk) clk->mark(PH_BND);
  rec(st->ev_jg, G);
  rec(st->ev_jc, C);
  wait(M, st->ev_jg);
  wait(M, st->ev_jc);
  trace_flush(tr, ctx);
}

}  // namespace

mics_step* step_create(mics_ctx* ctx, const mics_step_cfg* cfg, bool settle) {
  if (!cfg || cfg->nlayers < 1 || !cfg->layer_params) raise(MICS_OUT_OF_RANGE, "step config needs >= 1 layer");
  // every layer gathers something: the fence positions of the gather chain
  // (enqueue_gathers) and the first gather's wait for the boundary count on it
  for (int l = 0; l < cfg->nlayers; ++l)
    if (cfg->layer_params[l] == 0) raise(MICS_OUT_OF_RANGE, "layer " + std::to_string(l) + " has no parameters");
  if (cfg->grad_t != MICS_F32 && cfg->grad_t != MICS_BF16) raise(MICS_TYPE_MISMATCH, "gradients must be f32 or bf16");
  if (cfg->hier_k > 0) {
    if (!mics_partition_shape_ok(cfg->p, cfg->hier_k) || ctx->n % cfg->hier_k)
      raise(MICS_SHAPE_ERROR, "partition size p=" + std::to_string(cfg->p) + " is not node-aligned for k=" +
                                  std::to_string(cfg->hier_k));
  }
  auto* st = new mics_step();
  try {
    st->ctx = ctx;
    st->cfg = *cfg;
    st->layers.assign(cfg->layer_params, cfg->layer_params + cfg->nlayers);
    st->cfg.layer_params = nullptr;
    st->sync = sync_create(ctx, cfg->p, cfg->s, cfg->nlayers, st->layers.data(), MICS_F32, kAlignElems);
    mics_sync* sy = st->sync;
    const uint64_t S = sy->shard_elems, szg = dtype_size(cfg->grad_t);
    uint64_t maxl = 0;
    for (uint64_t c : sy->chunk) maxl = std::max(maxl, c * uint64_t(sy->p) * 2);
    st->gathered_half = round_up(maxl, 256);
    st->pbf16 = alloc_sym(ctx, S * 2);
    st->master = alloc_sym(ctx, S * 4);
    st->m = alloc_sym(ctx, S * 4);
    st->v = alloc_sym(ctx, S * 4);
    // Without compute nothing consumes a gather, so up to three run concurrently
    // (enqueue_gathers): three slots.  With compute a layer's GEMMs release its slot.
    const bool hier = cfg->hier_k > 0 && cfg->p > cfg->hier_k;
    const char* hme = std::getenv("MICS_HIER_MERGE");  // 0: one k_hier launch per visit (A/B runs)
    const bool hmerge = hier && !cfg->compute && !(hme && hme[0] == '0');
    // merged hierarchical launches take hier_group layer visits each (MICS_HIER_VISITS);
    // C4 all-gather phase on 4 B200 (n=8 / n=4 ranks), G = 1..4: 26.7/39.0, 25.9/35.5,
    // 25.5/34.7, 26.6/33.9 ms (profiles/r2/logs/R2q_*)
    st->hier_group = 3;
    if (const char* e = std::getenv("MICS_HIER_VISITS")) st->hier_group = std::max(1, std::min(4, std::atoi(e)));
    st->gather_slots = cfg->compute ? 2 : hmerge ? 3 * st->hier_group : 3;
    if (const char* e = std::getenv("MICS_GATHER_SLOTS"); e && !cfg->compute && !hmerge)
      st->gather_slots = std::max(3, std::min(kMaxGatherSlots, std::atoi(e)));
    st->gathered = alloc_sym(ctx, uint64_t(st->gather_slots) * st->gathered_half);
    // gradient slots: s resident sets, 1 regenerated per micro-step, or with compute 2
    // (the GEMMs of micro-step t+1 write one while the reduce-scatter of t reads the other)
    st->compute = cfg->compute != 0;
    st->gslots = st->compute ? std::min(2, cfg->s) : cfg->resident_grads ? cfg->s : 1;
    if (st->compute && (cfg->alternative || cfg->tokens == 0 || cfg->hidden == 0 || cfg->hidden % 8 || cfg->tokens % 8))
      raise(MICS_CONFIG_ERROR, "step with compute: 2-hop schedule, tokens and hidden multiples of 8");
    st->grads = alloc_sym(ctx, uint64_t(st->gslots) * sy->grad_elems * szg);
    // initial state: master = generator(seed ^ 0x5eed, "rank" = partition position r % p, layer 255),
    // so every replica of a shard starts identical; m = v = 0; bf16 copy of master
    for (int r = 0; r < ctx->n; ++r) {
      if (!ctx->local(r)) continue;
      launch_generate(ctx->stream, ctx->rank_ptr(st->master, r), MICS_F32, cfg->seed ^ 0x5eedull, r % cfg->p, 0, 255,
                      0, S, ctx->nsm * 8);
      MICS_CUDA(cudaMemsetAsync(ctx->rank_ptr(st->m, r), 0, S * 4, ctx->stream));
      MICS_CUDA(cudaMemsetAsync(ctx->rank_ptr(st->v, r), 0, S * 4, ctx->stream));
      launch_cast_bf16(ctx->stream, reinterpret_cast<const float*>(ctx->rank_ptr(st->master, r)),
                       reinterpret_cast<uint16_t*>(ctx->rank_ptr(st->pbf16, r)), S, ctx->nsm * 8);
    }
    if (st->compute) {
      for (int r = 0; r < ctx->n; ++r)  // padding past E_l stays zero: the GEMMs write [0, E_l) per layer
        if (ctx->local(r))
          MICS_CUDA(cudaMemsetAsync(ctx->rank_ptr(st->grads, r), 0, st->grads.stride, ctx->stream));
    } else if (cfg->resident_grads) {
      for (int t = 0; t < cfg->s; ++t) enqueue_generate(st, t);
    }
    // plans
    if (hier) {  // stage-1 tile flags of the hierarchical gathers
      uint64_t cmax = 0;
      for (uint64_t c : sy->chunk) cmax = std::max(cmax, c * 2);
      st->hflag_tiles = hier_flag_tiles(cmax);
      st->hflags = alloc_sym(ctx, uint64_t(cfg->p / cfg->hier_k) * st->hflag_tiles * 8);
      MICS_CUDA(cudaMemsetAsync(ctx->base + st->hflags.offset, 0, st->hflags.stride * uint64_t(ctx->per), ctx->stream));
    }
    for (int l = 0; l < cfg->nlayers; ++l) st->ag.push_back(build_layer_ag(st, l, cfg->compute ? 1 : 0));
    if (hmerge) build_hier_merged(st);
    for (int t = 0; t < cfg->s; ++t) {
      const uint64_t goff = uint64_t(t % st->gslots) * sy->grad_elems * szg;
      const int mode = t == 0 ? MICS_RS_ZERO_ACCUM : MICS_RS_ACCUMULATE;
      if (cfg->alternative)  // DeepSpeed default (sync_schedule.hpp:189-224): all-reduce over all n
        st->micro.push_back(build_alt(sy, st->grads, goff, cfg->grad_t, 1.0, true, mode));
      else  // 2-hop hop 1: reduce-scatter inside the partition group
        st->micro.push_back({build_micro_launch(sy, st->grads, goff, cfg->grad_t, 1.0, mode, true, false, 1, 1)});
    }
    st->adam.lr = cfg->lr;
    st->adam.beta1 = cfg->beta1;
    st->adam.beta2 = cfg->beta2;
    st->adam.eps = cfg->eps;
    st->adam.weight_decay = cfg->weight_decay;
    st->adam.step = 1;
    st->adam.grad_scale = 1.0 / (double(ctx->n) * cfg->s);  // mean over the global batch of n*s micro-batches
    st->adam.param = st->master;
    st->adam.exp_avg = st->m;
    st->adam.exp_avg_sq = st->v;
    st->adam.param_bf16 = st->pbf16;
    st->adam.write_grad = 0;
    if (!cfg->alternative) {
      st->bnd = build_boundary(sy, &st->adam, true, false);
      // overlapped tail (MICS_TAIL_OVERLAP=0/1 forces it)
      const char* te = std::getenv("MICS_TAIL_OVERLAP");
      // auto: any multi-process job with a replication fold (measured: N=2 17.48 -> 16.74 ms,
      // N=4 9.11 -> 8.96, one rank per GPU on 4 GPUs 9.94 -> 9.84)
      const bool auto_on = ctx->world > 1 && sy->n / sy->p > 1;
      st->tail = !st->compute && sy->n / sy->p > 1 && (te ? te[0] == '1' : auto_on);
      if (st->tail) {
        // K9 (default; MICS_TAIL_FUSED=0: the two-kernel boundary): each group's boundary
        // reduce-scatter and Adam in one launch, Adam blocks pulling a slice block as soon
        // as its owner published it, on channel 2
        const char* tfe = std::getenv("MICS_TAIL_FUSED");
        const bool fused_bnd = !(tfe && tfe[0] == '0') && sy->n / sy->p <= kTailMaxR;
        // two-kernel boundary: 8 groups when the last reduce-scatter stays inside a GPU
        // (HBM): N=2 16.36 -> 16.00 ms, N=4 8.68 -> 8.50; 4 when it crosses GPUs too (one
        // rank per GPU: 9.85 vs 10.39 ms at 8).  K9: 2 groups (fewer launch drains; C3
        // N=2 15.03 / N=4 8.81 ms at 2 groups vs 15.09 / 8.82 at 8)
        const char* tg = std::getenv("MICS_TAIL_GROUPS");  // experiments
        plan_layer_groups(st, tg ? std::max(1, std::atoi(tg)) : fused_bnd ? 2 : ctx->per >= cfg->p ? 8 : 4);
        const int s_last = cfg->s - 1;
        const uint64_t goff = uint64_t(s_last % st->gslots) * sy->grad_elems * szg;
        for (size_t g = 0; g < st->group_range.size(); ++g) {
          const int l0 = st->group_first_layer[g];
          const int l1 = g + 1 < st->group_first_layer.size() ? st->group_first_layer[g + 1] : cfg->nlayers;
          st->tail_rs.push_back(build_micro_launch(sy, st->grads, goff, cfg->grad_t, 1.0,
                                                   s_last == 0 ? MICS_RS_ZERO_ACCUM : MICS_RS_ACCUMULATE, true, false,
                                                   1, 1, nullptr, l0, l1));
          // boundary reduce-scatter on channel 2 (its own stream), Adam on channel 1 (side stream)
          if (!fused_bnd)
            st->tail_bnd.push_back(build_boundary_range(sy, &st->adam, sy->shard, st->group_range[g].first,
                                                      st->group_range[g].second, 1, 2));
        }
        if (fused_bnd) {
          const int r = sy->n / sy->p;
          uint32_t nblk_max = 1;
          for (const auto& [lo, hi] : st->group_range)
            nblk_max = std::max<uint32_t>(nblk_max, uint32_t(ceil_div(ceil_div(hi - lo, uint64_t(r)), fb_block())));
          const int G = int(st->group_range.size());
          st->fbflags = alloc_sym(ctx, (uint64_t(G) * uint64_t(r) * nblk_max + uint64_t(G)) * 8);
          MICS_CUDA(cudaMemsetAsync(ctx->base + st->fbflags.offset, 0, st->fbflags.stride * uint64_t(ctx->per),
                                    ctx->stream));
          for (int g = 0; g < G; ++g)
            st->tail_fb.push_back(build_boundary_fused_range(sy, &st->adam, st->group_range[size_t(g)].first,
                                                             st->group_range[size_t(g)].second, st->fbflags, g,
                                                             G, nblk_max, 2));
        }
        st->ev_tail.resize(st->group_range.size());
        for (auto& e : st->ev_tail) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        st->ev_tail_rs.resize(st->group_range.size());
        for (auto& e : st->ev_tail_rs) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        MICS_CUDA(cudaStreamCreateWithFlags(&st->tail_rs_stream, cudaStreamNonBlocking));
        MICS_CUDA(cudaEventCreateWithFlags(&st->ev_tail_done, cudaEventDisableTiming));

      }
      const char* fe = std::getenv("MICS_FUSED_TAIL");
      if (!st->tail && !st->compute && ctx->world == 1 && !(fe && fe[0] == '0') &&
          tail_supported(cfg->grad_t, sy->n / sy->p, sy->p))
        build_fused_tail(st);
    } else {  // shards already hold the global sum: the boundary is Adam on the own shard
      AdamPlan ap;
      uint64_t pmask = 0;
      for (int g = 0; g < sy->n / sy->p; ++g) {
        std::vector<int> ranks(static_cast<size_t>(sy->p));
        for (int i = 0; i < sy->p; ++i) ranks[size_t(i)] = g * sy->p + i;
        pmask |= ctx->peer_mask(ranks.data(), sy->p);
      }
      for (int r = 0; r < ctx->n; ++r) {
        if (!ctx->local(r)) continue;
        ap.add({ctx->rank_ptr(sy->shard, r)}, reinterpret_cast<float*>(ctx->rank_ptr(st->master, r)),
               reinterpret_cast<float*>(ctx->rank_ptr(st->m, r)), reinterpret_cast<float*>(ctx->rank_ptr(st->v, r)),
               reinterpret_cast<uint16_t*>(ctx->rank_ptr(st->pbf16, r)), nullptr, S, round_up(S, 4));
      }
      st->bnd.ag = make_adam_launch(ctx, ap, make_adam_scalars(cfg->lr, cfg->beta1, cfg->beta2, cfg->eps,
                                                               cfg->weight_decay, 1, st->adam.grad_scale),
                                    ctx->barrier(pmask, 0, 1), true);
      st->bnd.has_ag = true;
    }
    if (st->compute) setup_compute(st);
    // stats (per rank per step), algorithmic bytes of SURVEY §8(d)
    const int p = sy->p, r = sy->n / p;
    uint64_t csum = 0;
    for (uint64_t c : sy->chunk) csum += c;
    st->stats.ag_bytes_in = 2ull * uint64_t(cfg->s) * uint64_t(p - 1) * csum * 2;
    st->stats.rs_bytes_in = uint64_t(cfg->s) * uint64_t(p - 1) * csum * szg;
    st->stats.ar_bytes_in = r > 1 ? 2ull * uint64_t(r - 1) * sy->sub * 4 : 0;
    st->stats.adam_hbm_bytes = S * 30;
    st->stats.gen_bytes = generated(st) ? uint64_t(cfg->s) * sy->grad_elems * szg : 0;
    st->stats.shard_elems = S;
    st->stats.gathered_max_bytes = maxl;
    st->stats.gather_slots = uint64_t(st->gather_slots);
    st->stats.gather_slot_bytes = st->gathered_half;
    st->stats.grad_elems = sy->grad_elems;
    // everybody's initial parameters are written before anyone gathers them (the members
    // of a multi-device context settle together, capi.cpp)
    if (settle) {
      MICS_CUDA(cudaStreamSynchronize(ctx->stream));
      barrier_all(ctx);
      MICS_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    // kernels and algorithmic bytes of one step on this process (enqueue() skips empty launches)
    auto runs = [](const Launch& x) -> uint64_t { return (x.ndesc || x.bar.mask) ? 1 : 0; };
    mics_step_stats& S2 = st->stats;
    if (!st->agm.empty()) {
      for (auto& x : st->agm) {  // one micro-step's merged launches
        S2.ag_launches += uint64_t(cfg->s) * runs(x);
        S2.ag_remote_bytes += uint64_t(cfg->s) * x.remote_bytes;
        S2.ag_hbm_bytes += uint64_t(cfg->s) * x.hbm_bytes;
      }
    } else {
      for (auto& v : st->ag)
        for (auto& x : v) {  // forward + backward pass, every micro-step
          S2.ag_launches += 2 * uint64_t(cfg->s) * runs(x);
          S2.ag_remote_bytes += 2 * uint64_t(cfg->s) * x.remote_bytes;
          S2.ag_hbm_bytes += 2 * uint64_t(cfg->s) * x.hbm_bytes;
        }
    }
    for (size_t t = 0; t < st->micro.size(); ++t) {
      if ((st->tail || st->fused_tail) && t + 1 == st->micro.size()) continue;  // replaced by the tail launches
      for (auto& x : st->micro[t]) {
        S2.rs_launches += runs(x);
        S2.rs_remote_bytes += x.remote_bytes;
        S2.rs_hbm_bytes += x.hbm_bytes;
      }
    }
    for (auto& x : st->tail_rs) {
      S2.rs_launches += runs(x);
      S2.rs_remote_bytes += x.remote_bytes;
      S2.rs_hbm_bytes += x.hbm_bytes;
    }
    std::vector<const BoundaryLaunches*> bl;
    if (st->tail && !st->tail_fb.empty()) {
      for (const auto& x : st->tail_fb) {
        S2.bnd_launches += runs(x);
        S2.bnd_remote_bytes += x.remote_bytes;
        S2.bnd_hbm_bytes += x.hbm_bytes;
      }
    } else if (st->tail)
      for (const auto& x : st->tail_bnd) bl.push_back(&x);
    else if (!st->fused_tail)
      bl.push_back(&st->bnd);
    if (st->fused_tail) {
      S2.bnd_launches += 1;
      S2.bnd_hbm_bytes += st->ftail.hbm_bytes;
      S2.bnd_remote_bytes += st->ftail.remote_bytes;
    }
    for (const BoundaryLaunches* b : bl)
      for (const Launch* x : {&b->rs, &b->ag}) {
        if ((x == &b->rs && !b->has_rs) || (x == &b->ag && !b->has_ag)) continue;
        S2.bnd_launches += runs(*x);
        S2.bnd_remote_bytes += x->remote_bytes;
        S2.bnd_hbm_bytes += x->hbm_bytes;
      }
    S2.launches = S2.ag_launches + S2.rs_launches + S2.bnd_launches +
                  (generated(st) ? uint64_t(cfg->s) * uint64_t(ctx->per) : 0);
    if (st->compute) {
      for (const auto* v : {&st->gfwd, &st->gdgrad, &st->gwgrad})
        for (const GemmLaunch& g : *v) {
          S2.compute_flops += g.flops;
          S2.gemm_launches++;
        }
      if (st->recompute)
        for (const GemmLaunch& g : st->gfwd) {
          S2.compute_flops += g.flops;
          S2.gemm_launches++;
        }
      S2.launches += S2.gemm_launches;
    }
  } catch (...) {
    release(st);
    delete st;
    throw;
  }
  return st;
}

void step_destroy(mics_step* st) {
  if (!st) return;
  cudaStreamSynchronize(st->ctx->stream);
  release(st);
  delete st->sync;
  delete st;
}

namespace {
bool graph_enabled(const mics_step* st) {
  const char* e = std::getenv("MICS_GRAPH");
  return !(e && e[0] == '0');
}

// Capture one whole step (s micro-steps + boundary) into a CUDA graph.  The
// boundary kernels read their per-step scalars from st->d_scalars, so the same
// graph replays every step; programmatic-dependent-launch edges are kept by the
// capture.  The capture itself launches nothing: the state it advanced (Adam
// step) is rolled back and re-advanced per replay.
void build_graph(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  st->graph_tried = true;
  MICS_CUDA(cudaMalloc(&st->d_scalars, sizeof(DevScalars)));
  st->bnd.rs.dyn = st->bnd.ag.dyn = st->d_scalars;
  for (auto& b : st->tail_bnd) b.ag.dyn = st->d_scalars;
  for (auto& l : st->tail_fb) l.dyn = st->d_scalars;
  st->ftail.dyn = st->d_scalars;
  const int adam_step0 = st->adam_step;
  const uint64_t fb_epoch0 = st->fb_epoch;
  const uint64_t launches0 = ctx->launches;
  cudaGraph_t g = nullptr;
  MICS_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  st->capturing = true;
  try {
    if (st->compute) {
      enqueue_compute_step(st, nullptr);
    } else {
      for (int t = 0; t < st->cfg.s; ++t) {
        if (generated(st)) enqueue_generate(st, t);
        if ((st->tail || st->fused_tail) && t == st->cfg.s - 1) {
          enqueue_gathers(st, t);
          if (st->tail)
            enqueue_tail(st, nullptr);
          else
            enqueue_fused_tail(st);
        } else {
          enqueue_micro(st, t);
        }
      }
      if (!st->tail && !st->fused_tail) enqueue_boundary(st);
    }
  } catch (...) {
    st->capturing = false;
    cudaStreamEndCapture(ctx->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  st->capturing = false;
  MICS_CUDA(cudaStreamEndCapture(ctx->stream, &g));
  if (st->compute) {
    // events recorded during the capture belong to the graph: eager steps (profile,
    // run_host) after it need events that were never captured
    for (cudaEvent_t* e : {&st->ev_g[0], &st->ev_g[1], &st->ev_free[0], &st->ev_free[1], &st->ev_fork, &st->ev_jg,
                           &st->ev_jc}) {
      MICS_CUDA(cudaEventDestroy(*e));
      MICS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    for (auto* v : {&st->ev_wg, &st->ev_rsd, &st->ev_copied})
      for (auto& e : *v) {
        MICS_CUDA(cudaEventDestroy(e));
        MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
  }
  st->graph_launches = ctx->launches - launches0;
  ctx->launches = launches0;
  st->adam_step = adam_step0;
  st->fb_epoch = fb_epoch0;
  const cudaError_t e = cudaGraphInstantiate(&st->gexec, g, 0);
  cudaGraphDestroy(g);
  MICS_CUDA(e);
}

void replay(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  st->adam_step++;
  DevScalars v{};
  v.sc = make_adam_scalars(st->cfg.lr, st->cfg.beta1, st->cfg.beta2, st->cfg.eps, st->cfg.weight_decay,
                           st->adam_step, st->adam.grad_scale);
  if (!st->tail_fb.empty()) v.epoch = ++st->fb_epoch;
  launch_set_scalars(ctx->stream, st->d_scalars, v);
  MICS_CUDA(cudaGraphLaunch(st->gexec, ctx->stream));
  ctx->launches += st->graph_launches + 1;
  st->step_idx++;
}
}  // namespace

void step_run(mics_step* st, int iters) {
  if (iters > 0 && graph_enabled(st)) {
    if (!st->graph_tried) build_graph(st);
    for (int it = 0; it < iters; ++it) replay(st);
    st->stats.adam_step = st->adam_step;
    return;
  }
  for (int it = 0; it < iters; ++it) {
    if (st->compute) {
      enqueue_compute_step(st, nullptr);
      st->step_idx++;
      continue;
    }
    for (int t = 0; t < st->cfg.s; ++t) {
      if (generated(st)) enqueue_generate(st, t);
      if ((st->tail || st->fused_tail) && t == st->cfg.s - 1) {
        enqueue_gathers(st, t);
        if (st->tail)
          enqueue_tail(st, nullptr);
        else
          enqueue_fused_tail(st);
      } else {
        enqueue_micro(st, t);
      }
    }
    if (!st->tail && !st->fused_tail) enqueue_boundary(st);
    st->step_idx++;
  }
  st->stats.adam_step = st->adam_step;
}

ProfileRec* step_profile_begin(mics_step* st) {
  mics_ctx* ctx = st->ctx;
  const int s = st->cfg.s;
  auto* rec = new ProfileRec();
  if (st->compute) {  // serialised on the main stream, events around every gather / GEMM group
    PhaseClock clk;
    clk.s = ctx->stream;
    enqueue_compute_step(st, &clk);
    st->step_idx++;
    rec->compute = true;
    rec->ev = std::move(clk.ev);
    rec->kind = std::move(clk.kind);
    return rec;
  }
  std::vector<cudaEvent_t>& ev = rec->ev;
  ev.resize(size_t(4 * s + 2));
  for (auto& e : ev) MICS_CUDA(cudaEventCreate(&e));
  int k = 0;
  for (int t = 0; t < s; ++t) {
    MICS_CUDA(cudaEventRecord(ev[size_t(k++)], ctx->stream));
    if (generated(st)) enqueue_generate(st, t);
    MICS_CUDA(cudaEventRecord(ev[size_t(k++)], ctx->stream));
    enqueue_gathers(st, t);
    MICS_CUDA(cudaEventRecord(ev[size_t(k++)], ctx->stream));
    if (!((st->tail || st->fused_tail) && t == s - 1)) enqueue_sync(st, t);
    MICS_CUDA(cudaEventRecord(ev[size_t(k++)], ctx->stream));
  }
  MICS_CUDA(cudaEventRecord(ev[size_t(k++)], ctx->stream));
  if (st->tail)  // overlapped tail, serialised: RS / boundary per layer group
    enqueue_tail(st, &rec->tclk);
  else if (st->fused_tail)
    enqueue_fused_tail(st);  // timed as the boundary phase (it carries the last reduce-scatter)
  else
    enqueue_boundary(st);
  st->step_idx++;
  MICS_CUDA(cudaEventRecord(ev[size_t(k++)], ctx->stream));
  return rec;
}

void step_profile_end(mics_step* st, ProfileRec* rec, double* ms) {
  const int s = st->cfg.s;
  for (int i = 0; i < 5; ++i) ms[i] = 0;
  std::vector<cudaEvent_t>& ev = rec->ev;
  MICS_CUDA(cudaEventSynchronize(ev.back()));
  if (rec->compute) {
    for (size_t i = 1; i < ev.size(); ++i) {
      float x = 0;
      MICS_CUDA(cudaEventElapsedTime(&x, ev[i - 1], ev[i]));
      if (rec->kind[i] >= 0) ms[rec->kind[i]] += x;
    }
  } else {
    float a = 0, r = 0, g = 0, b = 0, x;
    for (int t = 0; t < s; ++t) {
      MICS_CUDA(cudaEventElapsedTime(&x, ev[size_t(4 * t)], ev[size_t(4 * t + 1)]));
      g += x;
      MICS_CUDA(cudaEventElapsedTime(&x, ev[size_t(4 * t + 1)], ev[size_t(4 * t + 2)]));
      a += x;
      MICS_CUDA(cudaEventElapsedTime(&x, ev[size_t(4 * t + 2)], ev[size_t(4 * t + 3)]));
      r += x;
    }
    MICS_CUDA(cudaEventElapsedTime(&x, ev[size_t(4 * s)], ev[size_t(4 * s + 1)]));
    b = x;
    if (st->tail) {
      b = 0;
      for (size_t i = 1; i < rec->tclk.size(); ++i) {
        MICS_CUDA(cudaEventElapsedTime(&x, rec->tclk[i - 1], rec->tclk[i]));
        (i % 2 ? r : b) += x;
      }
    }
    ms[0] = a;
    ms[1] = r;
    ms[2] = b;
    ms[3] = g;
  }
  for (auto e : rec->tclk) cudaEventDestroy(e);
  for (auto e : ev) cudaEventDestroy(e);
  delete rec;
  st->stats.adam_step = st->adam_step;
}

// One step with CUDA events around each phase; milliseconds per phase (ms[0] all-gather,
// [1] reduce-scatter, [2] boundary, [3] generation, [4] GEMMs).
void step_profile(mics_step* st, double* ms) { step_profile_end(st, step_profile_begin(st), ms); }

// End-to-end variant through host memory: every micro-step each local rank's
// gradients are copied from (pinned) host memory — host_grads holds one gradient
// set of grad_elems, reused for every local rank and micro-step (one DMA each) —
// and after the boundary a fixed-size slice of every local rank's updated master
// shard is read back.
void step_run_host(mics_step* st, const void* host_grads, int iters, void* host_result) {
  mics_ctx* ctx = st->ctx;
  const uint64_t szg = dtype_size(st->cfg.grad_t), gb = st->sync->grad_elems * szg;
  const uint64_t rb = std::min(st->host_result_elems, st->sync->shard_elems) * 4;
  if (st->compute) {  // inputs X of every micro-step and local rank (tokens x hidden bf16), then the step
    const uint64_t xb = st->T * st->h * 2;
    const uint64_t rb = std::min(st->host_result_elems, st->sync->shard_elems) * 4;
    for (int it = 0; it < iters; ++it) {
      for (int t = 0; t < st->cfg.s; ++t)
        for (int r = 0; r < ctx->n; ++r)
          if (ctx->local(r))
            MICS_CUDA(cudaMemcpyAsync(ctx->rank_ptr(st->x, r) + uint64_t(t) * xb, host_grads, xb,
                                      cudaMemcpyHostToDevice, ctx->stream));
      enqueue_compute_step(st, nullptr);
      st->step_idx++;
      if (host_result) {
        int li = 0;
        for (int r = 0; r < ctx->n; ++r)
          if (ctx->local(r))
            MICS_CUDA(cudaMemcpyAsync(static_cast<char*>(host_result) + uint64_t(li++) * rb,
                                      ctx->rank_ptr(st->master, r), rb, cudaMemcpyDeviceToHost, ctx->stream));
      }
    }
    st->stats.adam_step = st->adam_step;
    return;
  }
  const int s = st->cfg.s, nslot = st->gslots;
  if (!st->copy_stream) {
    MICS_CUDA(cudaStreamCreateWithFlags(&st->copy_stream, cudaStreamNonBlocking));
    st->ev_h2d.resize(size_t(nslot));
    st->ev_rs_slot.resize(size_t(nslot));
    for (auto& e : st->ev_h2d) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : st->ev_rs_slot) MICS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MICS_CUDA(cudaEventCreateWithFlags(&st->ev_begin, cudaEventDisableTiming));
  }
  // slot k's copy waits until the reduce-scatter that last read slot k is done
  auto copy_in = [&](int t) {
    const int k = t % nslot;
    MICS_CUDA(cudaStreamWaitEvent(st->copy_stream, st->ev_rs_slot[size_t(k)], 0));
    for (int r = 0; r < ctx->n; ++r) {
      if (!ctx->local(r)) continue;
      MICS_CUDA(cudaMemcpyAsync(ctx->rank_ptr(st->grads, r) + uint64_t(k) * gb, host_grads, gb,
                                cudaMemcpyHostToDevice, st->copy_stream));
    }
    MICS_CUDA(cudaEventRecord(st->ev_h2d[size_t(k)], st->copy_stream));
  };
  // nothing of this call starts before the work already on the main stream (e.g. a timing event)
  MICS_CUDA(cudaEventRecord(st->ev_begin, ctx->stream));
  MICS_CUDA(cudaStreamWaitEvent(st->copy_stream, st->ev_begin, 0));
  for (int it = 0; it < iters; ++it) {
    // resident slots: every copy of the step can start at once (each waits only for
    // its own slot's previous reader); one slot: copy t+1 follows the RS of t
    if (nslot == s)
      for (int t = 0; t < s; ++t) copy_in(t);
    else
      copy_in(0);
    for (int t = 0; t < s; ++t) {
      const int k = t % nslot;
      enqueue_gathers(st, t);  // parameters only: overlaps the copies
      MICS_CUDA(cudaStreamWaitEvent(ctx->stream, st->ev_h2d[size_t(k)], 0));
      if (st->tail && t == s - 1)
        enqueue_tail(st, nullptr);  // last reduce-scatter + boundary, overlapped per layer group
      else if (st->fused_tail && t == s - 1)
        enqueue_fused_tail(st);     // last reduce-scatter + boundary + Adam in one kernel
      else
        enqueue_sync(st, t);
      MICS_CUDA(cudaEventRecord(st->ev_rs_slot[size_t(k)], ctx->stream));
      if (nslot != s && t + 1 < s) copy_in(t + 1);
    }
    if (!st->tail && !st->fused_tail) enqueue_boundary(st);
    st->step_idx++;
    if (host_result) {
      int li = 0;
      for (int r = 0; r < ctx->n; ++r) {
        if (!ctx->local(r)) continue;
        MICS_CUDA(cudaMemcpyAsync(static_cast<char*>(host_result) + uint64_t(li) * rb, ctx->rank_ptr(st->master, r), rb,
                                  cudaMemcpyDeviceToHost, ctx->stream));
        ++li;
      }
    }
  }
  st->stats.adam_step = st->adam_step;
}

}  // namespace mics
