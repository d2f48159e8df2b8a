// Sync-state and step-driver internals shared by sync.cpp, step.cpp and capi.cpp.
#pragma once

#include <array>
#include <vector>

#include "internal.h"

struct mics_sync {
  // a multi-device context's sync state: one member state per GPU (capi.cpp runs every
  // call on each; queries read member 0 — the members evolve identically)
  std::vector<mics_sync*> subs;
  mics_ctx* ctx = nullptr;
  int n = 0, p = 0, s = 1, nseg = 0;
  mics_dtype acc_t = MICS_F32;
  std::vector<uint64_t> len, chunk, shard_off, grad_off;
  uint64_t shard_elems = 0, grad_elems = 0, sub = 0;
  mics_buf shard{};
  int micro_step = 0;
  std::vector<std::array<int64_t, 4>> events;
  // alternative schedule scratch (lazily allocated)
  bool alt_ready = false;
  mics_buf alt{};
  std::vector<uint64_t> alt_sub, alt_off;
};

namespace mics {

struct BoundaryLaunches {
  Launch rs, ag;
  bool has_rs = false, has_ag = false;
};

mics_buf alloc_sym(mics_ctx* c, uint64_t bytes_per_rank);
void barrier_all(mics_ctx* c);
void check_buf_rank(const mics_ctx* c, mics_buf b, int rank, uint64_t off, uint64_t bytes);

mics_sync* sync_create(mics_ctx* ctx, int p, int s, int nseg, const uint64_t* seg_len, mics_dtype acc_t,
                       uint32_t align);
Launch build_micro_launch(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale, int mode,
                          bool persistent, bool record, int entry, int exit,
                          const mics_buf* shard_override = nullptr, int seg_lo = 0, int seg_hi = -1);
BoundaryLaunches build_boundary(mics_sync* st, const mics_adam* adam, bool persistent, bool record);
BoundaryLaunches build_boundary_range(mics_sync* st, const mics_adam* adam, mics_buf shard, uint64_t lo, uint64_t hi,
                                      int chan, int rs_chan = -1);
// K9: layer group g of G; flags = per rank [G][r][nblk_max] u64 block flags, then G item tickets
Launch build_boundary_fused_range(mics_sync* st, const mics_adam* adam, uint64_t lo, uint64_t hi, mics_buf flags,
                                  int g, int G, uint32_t nblk_max, int chan);
void micro_step(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale, int mode);
void boundary(mics_sync* st, const mics_adam* adam);
void alt_step(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale);
std::vector<Launch> build_alt(mics_sync* st, mics_buf grads, uint64_t goff, mics_dtype grad_t, double scale,
                              bool persistent, int acc_mode);
void alt_boundary(mics_sync* st);

}  // namespace mics

// MiCS step driver state (step.cpp)
constexpr int kMaxGatherSlots = 12;  // mics_step::gather_slots upper bound (3 x merged hierarchical visits)

namespace mics {
struct ProfileRec {  // one profiled step in flight (step_profile_begin / step_profile_end)
  bool compute = false;
  std::vector<cudaEvent_t> ev, tclk;
  std::vector<int> kind;  // step with compute: the phase of the interval ending at ev[i]
};
}  // namespace mics

struct mics_step {
  // a multi-device context's step: one member step per GPU, and the group view of their
  // sync states (owned here; the member states belong to the member steps)
  std::vector<mics_step*> subs;
  mics_sync* gsync = nullptr;
  mics_ctx* ctx = nullptr;
  mics_step_cfg cfg{};
  std::vector<uint64_t> layers;
  mics_sync* sync = nullptr;
  mics_buf pbf16{}, master{}, m{}, v{}, gathered{}, grads{};
  uint64_t gathered_half = 0;                 // bytes of one gathered buffer (slot)
  int gather_slots = 2;                       // layer l gathers into slot l % gather_slots
  std::vector<std::vector<mics::Launch>> ag;  // per layer: 1 launch (k_copy flat or k_hier)
  // merged hierarchical gathers of one micro-step (comm-only step): 2L/G+1 k_hier launches
  std::vector<mics::Launch> agm;
  int hier_group = 3;  // G: layer visits per merged launch
  // hierarchical gathers (k_hier): per rank [q][hflag_tiles] u64 stage-1 tile flags
  mics_buf hflags{};
  uint64_t hflag_tiles = 0;
  // per micro-step: the 2-hop reduce-scatter, or the alternative schedule's
  // all-n reduce-scatter + all-gather + owned-chunk accumulate
  std::vector<std::vector<mics::Launch>> micro;
  mics::BoundaryLaunches bnd;
  mics_adam adam{};
  int adam_step = 0;
  mics_step_stats stats{};
  uint64_t host_result_elems = 4096;
  std::vector<std::pair<uint64_t, uint64_t>> group_range;  // shard range of each tail layer group
  std::vector<int> group_first_layer;
  uint64_t step_idx = 0;
  // Overlapped tail (2-hop, partition groups inside a GPU, replication groups across
  // GPUs — N=2/4 of the 8-rank job): the last micro-step's reduce-scatter (HBM) runs
  // per layer group on the main stream (channel 0) while each finished group's
  // boundary all-reduce + Adam (NVLink) runs on the side stream (channel 1).
  bool tail = false;
  // Fused tail (every rank on this GPU, N=1; MICS_FUSED_TAIL=0 disables): the last
  // micro-step's reduce-scatter + the boundary all-reduce + Adam as one K8 launch
  bool fused_tail = false;
  mics::Launch ftail{};
  std::vector<mics::Launch> tail_rs;
  std::vector<mics::BoundaryLaunches> tail_bnd;
  // K9 (default): each layer group's boundary as one fused launch (tail_bnd kept for A/B)
  std::vector<mics::Launch> tail_fb;
  mics_buf fbflags{};        // per rank [groups][r][nblk] u64 block flags
  uint64_t fb_epoch = 0;     // flag value of the current step
  std::vector<cudaEvent_t> ev_tail, ev_tail_rs;   // [group]: last RS done / boundary RS done
  cudaEvent_t ev_tail_done = nullptr;
  cudaStream_t tail_rs_stream = nullptr;          // boundary reduce-scatters (channel 2), ahead of Adam
  // CUDA-graph replay (default; MICS_GRAPH=0 enqueues every kernel per step):
  // one captured step whose boundary kernels read the per-step Adam scalars from
  // d_scalars, set by one small kernel before each replay.
  bool graph_tried = false, capturing = false;
  cudaGraphExec_t gexec = nullptr;
  mics::DevScalars* d_scalars = nullptr;
  uint64_t graph_launches = 0;  // kernels in one replay (the capture's count)
  // e2e (host gradients): H2D copies run on their own stream, one slot ahead of
  // the reduce-scatter that consumes them, overlapping the gathers
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_rs_slot;
  cudaEvent_t ev_begin = nullptr;
  // ---- step with compute (cfg.compute): layer l is W_l = gathered[0, E_l) viewed as
  // [rows_l = E_l / h, h]; X [T, h] per rank and micro-step slot; Y_l [T, ldy_l] stored
  // (or one recomputed scratch); dX [T, h] fp32.  Three streams: gathers (gs), GEMMs
  // (cs) and the reduce-scatters + boundary on ctx->stream, ordered by events.
  bool compute = false, recompute = false;
  uint64_t T = 0, h = 0;
  std::vector<uint64_t> rows, ldy, yoff;
  mics_buf x{}, y{}, dx{};
  int gslots = 1;                                    // gradient slots (micro-step t -> t % gslots)
  int comm_sms = 0;                                  // SMs left to the overlapped collectives (GEMMs get the rest)
  bool rs_overlap = true;                            // micro-step RS under the next micro-step's GEMMs
  std::vector<int> ag_grid_full, micro_grid_full;    // grids of the serialised (profile) step
  // flat gathers of the step with compute (MICS_CE_GATHER, default on): the
  // overlapped per-layer gathers are copy-engine memcpys (no SM time) instead of
  // k_copy: per layer, the (dst, src, bytes) of every local rank's p chunks
  bool ce_gather = false;
  struct CeCopy {
    void* dst;
    const void* src;
    uint64_t bytes;
  };
  std::vector<std::vector<CeCopy>> ce;
  // Copy-engine-staged reduce-scatter (step with compute, partition groups spanning
  // GPUs; MICS_CE_RS): the reduce-scatter of micro-step t (t < s-1) is carried by the
  // backward pass of t+1: on the gather stream, after each layer's gather, the copy
  // engines pull that layer's chunks of the peers' micro-step-t gradients into local
  // staging (between two barriers with the partition peers on channel 2), then
  // rs_local folds local + staged sources (HBM only, same fold order).  The last
  // micro-step, which overlaps nothing, keeps the SM pull reduce-scatter.
  bool ce_rs = false;
  mics_buf stage{};                              // per rank: [p][sum_l c_l] gradient dtype
  std::vector<std::vector<std::vector<CeCopy>>> ce_rs_copies;  // [slot][layer]
  std::vector<mics::Launch> rs_local;             // [micro-step]
  mics::Launch rs_bar{};                          // full barrier with the partition peers, channel 2
  std::vector<cudaEvent_t> ev_copied;             // [slot]
  std::vector<mics::GemmLaunch> gfwd, gdgrad, gwgrad;  // [(t * L + l) * per + local rank]
  cudaStream_t gs = nullptr, cs = nullptr;
  cudaEvent_t ev_g[2] = {}, ev_free[2] = {}, ev_fork = nullptr, ev_jg = nullptr, ev_jc = nullptr;
  std::vector<cudaEvent_t> ev_wg, ev_rsd;
};
