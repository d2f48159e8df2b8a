// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C shim over the UNMODIFIED reference hot path (sdpsim), compiled straight
// from /root/reference/proj/src/{topology,collectives}.cpp plus the
// header-only sync_schedule.hpp by oracle/Makefile into oracle/_ref/.
// Used by tests/golden/make_golden.py to produce golden vectors, by the
// CPU parity tests (when present) and by bench.py's cpu_baseline /
// `--impl reference` leg.  Each entry point names the reference symbol it
// wraps.  Reference exceptions (sdpsim::Error, errors.hpp:22-34) are mapped
// to 1 + Errc ordinal with the message kept in ref_last_error().
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "sdpsim/collectives.hpp"
#include "sdpsim/sync_schedule.hpp"
#include "sdpsim/topology.hpp"

using namespace sdpsim;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

void dump_traffic(const VirtualRankEngine& eng, int64_t* traffic, int cap, int* ntraffic) {
  if (!ntraffic) return;
  auto t = eng.traffic();
  int i = 0;
  for (const auto& [key, bytes] : t) {
    if (traffic && i < cap) {
      traffic[3 * i + 0] = key.first;
      traffic[3 * i + 1] = key.second;
      traffic[3 * i + 2] = static_cast<int64_t>(bytes);
    }
    ++i;
  }
  *ntraffic = i;
}

std::vector<Bytes> split(const uint8_t* data, int count, size_t each) {
  std::vector<Bytes> out(count);
  for (int i = 0; i < count; ++i) {
    out[i].resize(each);
    if (each) std::memcpy(out[i].data(), data + i * each, each);
  }
  return out;
}

void join(const std::vector<Bytes>& v, uint8_t* out) {
  size_t off = 0;
  for (const auto& b : v) {
    if (!b.empty()) std::memcpy(out + off, b.data(), b.size());
    off += b.size();
  }
}

CollectiveGroup make_group(const int* ranks, int p) {
  CollectiveGroup g;
  g.ranks.assign(ranks, ranks + p);
  return g;
}

DType to_dtype(int d) {
  switch (d) {
    case 0: return DType::i64;
    case 1: return DType::f32;
    default: return DType::f64;
  }
}

template <typename T>
std::vector<std::vector<std::vector<T>>> unpack_grads(const T* g, int s, int n, size_t len) {
  std::vector<std::vector<std::vector<T>>> out(s, std::vector<std::vector<T>>(n));
  for (int t = 0; t < s; ++t)
    for (int r = 0; r < n; ++r) out[t][r].assign(g + (size_t(t) * n + r) * len, g + (size_t(t) * n + r + 1) * len);
  return out;
}

void dump_events(const std::vector<SyncEvent>& log, int64_t* ev, int cap, int* nev) {
  if (!nev) return;
  int i = 0;
  for (const auto& e : log) {
    if (ev && i < cap) {
      ev[4 * i + 0] = e.step;
      ev[4 * i + 1] = static_cast<int64_t>(e.phase);
      ev[4 * i + 2] = e.group_id;
      ev[4 * i + 3] = static_cast<int64_t>(e.bytes);
    }
    ++i;
  }
  *nev = i;
}

// mode 0 = two-hop (sync_schedule.hpp:118-185), 1 = alternative (:189-232),
// 2 = oracle_global_sync (:236-256).
template <typename T>
int run_schedule(int mode, int threads, int n, int p, int s, size_t len, const T* grads, T* out,
                 int64_t* ev, int cap, int* nev, int64_t* traffic, int tcap, int* ntraffic) {
  return guarded([&] {
    GroupLayout layout = build_group_layout(n, p);
    auto g = unpack_grads(grads, s, n, len);
    const size_t chunk = owned_chunk_elems(layout, len);
    VirtualRankEngine engine(threads);
    std::vector<SyncEvent> log;
    std::vector<std::vector<T>> result(n);
    if (mode == 2) {
      result = oracle_global_sync(g, layout);
    } else {
      auto st = make_sync_states<T>(layout, len, s);
      for (int t = 0; t < s; ++t) {
        if (mode == 0)
          two_hop_micro_step(engine, layout, st, g[t], &log);
        else
          alternative_schedule_step(engine, layout, st, g[t], &log);
      }
      if (mode == 0)
        two_hop_boundary(engine, layout, st, &log);
      else
        alternative_boundary(st);
      for (int r = 0; r < n; ++r) result[r] = st[r].shard;
    }
    for (int r = 0; r < n; ++r) std::memcpy(out + size_t(r) * chunk, result[r].data(), chunk * sizeof(T));
    dump_events(log, ev, cap, nev);
    dump_traffic(engine, traffic, tcap, ntraffic);
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- generators used by the reference tests (test_collectives.cpp:13-21,
// test_sync_schedule.cpp:13-28, acceptance_main.cpp:37-45, sdpsim_main.cpp:132-140)
void ref_random_shards(int count, size_t chunk, uint32_t seed, uint8_t* out) {
  std::mt19937 rng(seed);
  for (size_t i = 0; i < size_t(count) * chunk; ++i) out[i] = static_cast<uint8_t>(rng() & 0xff);
}
void ref_random_i64(size_t count, int64_t lo, int64_t hi, uint32_t seed, int64_t* out) {
  std::mt19937 rng(seed);
  std::uniform_int_distribution<std::int64_t> d(lo, hi);
  for (size_t i = 0; i < count; ++i) out[i] = d(rng);
}
void ref_random_f32(size_t count, float lo, float hi, uint32_t seed, float* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<float> d(lo, hi);
  for (size_t i = 0; i < count; ++i) out[i] = d(rng);
}

// ---- topology (topology.cpp)
int ref_build_group_layout(int n, int p, int* part, int* repl) {
  return guarded([&] {
    GroupLayout l = build_group_layout(n, p);
    int i = 0;
    for (const auto& g : l.partition_groups)
      for (int r : g) part[i++] = r;
    i = 0;
    for (const auto& g : l.replication_groups)
      for (int r : g) repl[i++] = r;
  });
}
int ref_partition_shape_ok(int p, int k) { return partition_shape_ok(p, k) ? 1 : 0; }
int ref_model_state_bytes(uint64_t params, uint64_t bpp, uint64_t* out) {
  return guarded([&] { *out = model_state_bytes(params, bpp); });
}
int ref_cluster_validate(int num_nodes, int k, double intra, double inter, double a_intra, double a_inter) {
  return guarded([&] {
    ClusterSpec c;
    c.num_nodes = num_nodes;
    c.devices_per_node = k;
    c.intra_node_bandwidth = intra;
    c.inter_node_bandwidth_per_node = inter;
    c.alpha_intra = a_intra;
    c.alpha_inter = a_inter;
    c.validate();
  });
}
int ref_min_feasible_partition(uint64_t states, int num_nodes, int k, uint64_t device_memory,
                               int node_granular, double headroom, int* out) {
  return guarded([&] {
    ClusterSpec c;
    c.num_nodes = num_nodes;
    c.devices_per_node = k;
    c.intra_node_bandwidth = 1;
    c.inter_node_bandwidth_per_node = 1;
    c.device_memory = device_memory;
    *out = min_feasible_partition(states, c, node_granular != 0, headroom);
  });
}

// ---- collectives (collectives.cpp:103-321)
int ref_all_gather(int threads, const int* ranks, int p, const uint8_t* shards, size_t chunk, uint8_t* out,
                   int64_t* traffic, int tcap, int* ntraffic) {
  return guarded([&] {
    VirtualRankEngine engine(threads);
    auto res = all_gather(engine, make_group(ranks, p), split(shards, p, chunk));
    join(res, out);
    dump_traffic(engine, traffic, tcap, ntraffic);
  });
}

int ref_reduce_scatter(int threads, const int* ranks, int p, const uint8_t* bufs, size_t bytes, int dtype,
                       uint8_t* out, int64_t* traffic, int tcap, int* ntraffic) {
  return guarded([&] {
    VirtualRankEngine engine(threads);
    auto res = reduce_scatter(engine, make_group(ranks, p), split(bufs, p, bytes), to_dtype(dtype));
    join(res, out);
    dump_traffic(engine, traffic, tcap, ntraffic);
  });
}

int ref_all_reduce(int threads, const int* ranks, int p, const uint8_t* bufs, size_t bytes, int dtype,
                   uint8_t* out, int64_t* traffic, int tcap, int* ntraffic) {
  return guarded([&] {
    VirtualRankEngine engine(threads);
    auto res = all_reduce(engine, make_group(ranks, p), split(bufs, p, bytes), to_dtype(dtype));
    join(res, out);
    dump_traffic(engine, traffic, tcap, ntraffic);
  });
}

// Cluster as in test_collectives.cpp:102-106: num_nodes = n/k, k devices per node.
int ref_hier_all_gather(int threads, int n, int p, int k, const uint8_t* shards, size_t chunk, int corrupt,
                        uint8_t* out, int64_t* traffic, int tcap, int* ntraffic) {
  return guarded([&] {
    ClusterSpec cluster;
    cluster.num_nodes = n / k;
    cluster.devices_per_node = k;
    cluster.intra_node_bandwidth = 1;
    cluster.inter_node_bandwidth_per_node = 1;
    GroupLayout layout = build_group_layout(n, p);
    VirtualRankEngine engine(threads);
    HierarchicalOptions opts;
    opts.corrupt_stage2 = corrupt != 0;
    auto res = hierarchical_all_gather(engine, layout, cluster, split(shards, n, chunk), opts);
    join(res, out);
    dump_traffic(engine, traffic, tcap, ntraffic);
  });
}

// groups: `count` groups, sizes[b] ranks each (concatenated in `ranks`),
// group b's shards are sizes[b] x chunks[b] bytes concatenated in `shards`.
int ref_batched_all_gather(int threads, int count, const int* sizes, const int* ranks, const size_t* chunks,
                           const uint8_t* shards, uint8_t* out) {
  return guarded([&] {
    VirtualRankEngine engine(threads);
    std::vector<CollectiveGroup> groups;
    std::vector<std::vector<Bytes>> sets;
    size_t roff = 0, soff = 0;
    for (int b = 0; b < count; ++b) {
      groups.push_back(make_group(ranks + roff, sizes[b]));
      sets.push_back(split(shards + soff, sizes[b], chunks[b]));
      roff += sizes[b];
      soff += size_t(sizes[b]) * chunks[b];
    }
    auto res = batched_all_gather(engine, groups, sets);
    size_t ooff = 0;
    for (int b = 0; b < count; ++b) {
      join(res[b], out + ooff);
      ooff += size_t(sizes[b]) * sizes[b] * chunks[b];
    }
  });
}

int ref_batched_reduce_scatter(int threads, int count, const int* sizes, const int* ranks, const size_t* bytes,
                               const uint8_t* bufs, int dtype, uint8_t* out) {
  return guarded([&] {
    VirtualRankEngine engine(threads);
    std::vector<CollectiveGroup> groups;
    std::vector<std::vector<Bytes>> sets;
    size_t roff = 0, soff = 0;
    for (int b = 0; b < count; ++b) {
      groups.push_back(make_group(ranks + roff, sizes[b]));
      sets.push_back(split(bufs + soff, sizes[b], bytes[b]));
      roff += sizes[b];
      soff += size_t(sizes[b]) * bytes[b];
    }
    auto res = batched_reduce_scatter(engine, groups, sets, to_dtype(dtype));
    size_t ooff = 0;
    for (int b = 0; b < count; ++b) {
      join(res[b], out + ooff);
      ooff += bytes[b];  // p outputs of bytes/p each
    }
  });
}

// ---- sync schedule (sync_schedule.hpp). grads: s x n x len; out: n x chunk.
// events: 4 int64 per event (step, phase, group, bytes).
#define REF_SCHED(NAME, T, MODE)                                                                 \
  int NAME(int threads, int n, int p, int s, size_t len, const T* grads, T* out, int64_t* ev,   \
           int cap, int* nev, int64_t* traffic, int tcap, int* ntraffic) {                       \
    return run_schedule<T>(MODE, threads, n, p, s, len, grads, out, ev, cap, nev, traffic, tcap, \
                           ntraffic);                                                            \
  }
REF_SCHED(ref_two_hop_i64, int64_t, 0)
REF_SCHED(ref_two_hop_f32, float, 0)
REF_SCHED(ref_two_hop_f64, double, 0)
REF_SCHED(ref_alternative_i64, int64_t, 1)
REF_SCHED(ref_alternative_f32, float, 1)
REF_SCHED(ref_alternative_f64, double, 1)
REF_SCHED(ref_global_sync_i64, int64_t, 2)
REF_SCHED(ref_global_sync_f32, float, 2)
REF_SCHED(ref_global_sync_f64, double, 2)

// CPU baseline of one MiCS step over a bounded sample of layers, through the
// reference's own functions: per micro-step a per-layer parameter all_gather in
// every partition group (forward and backward pass, simulator.cpp:265-280 order),
// two_hop_micro_step over the sample's flat gradient, then two_hop_boundary.  The
// reference has no optimizer; the sharded Adam of the B200 step is
// added as a plain loop with the documented formula so both sides do the same
// work.  Inputs are built outside the timed region; returns the best of `reps`
// wall-clock seconds (std::chrono::steady_clock).
double ref_step_sample(int threads, int n, int p, int s, int nlayers, const uint64_t* layer_params, int reps) {
  double best = 1e300;
  try {
    GroupLayout layout = build_group_layout(n, p);
    uint64_t len = 0;
    for (int l = 0; l < nlayers; ++l) len += layer_params[l];
    std::mt19937 rng(2205);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    // bf16 parameter shards per layer per rank
    std::vector<std::vector<Bytes>> shards(static_cast<size_t>(nlayers));
    for (int l = 0; l < nlayers; ++l) {
      const size_t c = (layer_params[l] + p - 1) / p * 2;
      shards[size_t(l)].resize(size_t(n));
      for (auto& b : shards[size_t(l)]) {
        b.resize(c);
        for (auto& x : b) x = static_cast<std::byte>(rng() & 0xff);
      }
    }
    std::vector<std::vector<std::vector<float>>> grads(static_cast<size_t>(s),
                                                       std::vector<std::vector<float>>(static_cast<size_t>(n)));
    for (auto& st : grads)
      for (auto& g : st) {
        g.resize(len);
        for (auto& v : g) v = dist(rng);
      }
    const size_t chunk = owned_chunk_elems(layout, len);
    std::vector<float> param(chunk, 0.5f), m(chunk, 0.0f), v(chunk, 0.0f);
    for (int rep = 0; rep < reps; ++rep) {
      VirtualRankEngine engine(threads);
      auto states = make_sync_states<float>(layout, len, s);
      std::vector<std::vector<float>> P(size_t(n), param), M(size_t(n), m), V(size_t(n), v);
      const auto t0 = std::chrono::steady_clock::now();
      for (int t = 0; t < s; ++t) {
        for (int pass = 0; pass < 2; ++pass)
          for (int li = 0; li < nlayers; ++li) {
            const int l = pass == 0 ? li : nlayers - 1 - li;
            for (int g = 0; g < layout.num_partition_groups(); ++g) {
              CollectiveGroup grp{layout.partition_groups[size_t(g)]};
              std::vector<Bytes> in(shards[size_t(l)].begin() + g * p, shards[size_t(l)].begin() + (g + 1) * p);
              auto out = all_gather(engine, grp, in);
              (void)out;
            }
          }
        two_hop_micro_step(engine, layout, states, grads[size_t(t)]);
      }
      two_hop_boundary(engine, layout, states);
      const float b1 = 0.9f, b2 = 0.999f, omb1 = 0.1f, omb2 = 0.001f, eps = 1e-8f, ss = 1e-4f, bc2 = 0.0316f;
      const float gs = 1.0f / float(n * s);
      for (int r = 0; r < n; ++r) {
        const auto& gsh = states[size_t(r)].shard;
        for (size_t e = 0; e < chunk; ++e) {
          const float gg = gsh[e] * gs;
          M[size_t(r)][e] = b1 * M[size_t(r)][e] + omb1 * gg;
          V[size_t(r)][e] = b2 * V[size_t(r)][e] + omb2 * (gg * gg);
          P[size_t(r)][e] = P[size_t(r)][e] - ss * (M[size_t(r)][e] / (std::sqrt(V[size_t(r)][e]) / bc2 + eps));
        }
      }
      const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      best = std::min(best, sec);
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
  return best;
}

// State-machine probe (test_sync_schedule.cpp:117-132): runs `ops`, a string
// of 'm' (micro-step) / 'b' (boundary); returns per-op status in `codes`.
int ref_state_machine(int n, int p, int s, size_t len, const char* ops, int* codes) {
  GroupLayout layout = build_group_layout(n, p);
  VirtualRankEngine engine(1);
  auto st = make_sync_states<std::int64_t>(layout, len, s);
  std::vector<std::vector<std::int64_t>> grads(n, std::vector<std::int64_t>(len, 1));
  for (int i = 0; ops[i]; ++i) {
    codes[i] = guarded([&] {
      if (ops[i] == 'm')
        two_hop_micro_step(engine, layout, st, grads);
      else
        two_hop_boundary(engine, layout, st);
    });
  }
  return 0;
}

}  // extern "C"
