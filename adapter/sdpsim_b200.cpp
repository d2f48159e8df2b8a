// sdpsim -> libmics adapter: the reference's C++ API (the declarations in
// /root/reference/proj/include/sdpsim/{topology,collectives}.hpp, used in place,
// never copied) implemented by forwarding to the B200 C-ABI (include/mics.h).
//
// Linking the reference's own unit suites (proj/tests/test_topology.cpp,
// test_collectives.cpp, test_sync_schedule.cpp) against this file instead of
// proj/src/{topology,collectives}.cpp runs them on the GPU: every collective —
// including the ones inside the header-only 2-hop schedule templates — executes
// as libmics kernels on cuda:0.  This is the reference-side binding of
// INTEGRATION.md §2, exercised for real.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "mics.h"
#include "sdpsim/collectives.hpp"
#include "sdpsim/topology.hpp"

namespace sdpsim {

namespace {

[[noreturn]] void rethrow(mics_status s) {
  // mics_status = 1 + Errc ordinal; the message already reads "<Errc>: detail"
  const int code = int(s) - 1;
  const Errc e = code >= 0 && code <= int(Errc::ConfigError) ? Errc(code) : Errc::ConfigError;
  throw Error(e, mics_last_error());
}
void check(mics_status s) {
  if (s != MICS_OK) rethrow(s);
}

// One process-wide context: the reference's engines are in-process virtual ranks, so
// every VirtualRankEngine maps onto it.  MICS_DEVICES="0,1,..." spreads the ranks
// node-major over those GPUs of this process (mics_init_devices); default: GPU 0.
constexpr int kMaxRanks = 1024;
mics_ctx* ctx() {
  static mics_ctx* c = [] {
    mics_init_args a{kMaxRanks, 1, 0, 0, 2ull << 30};
    std::vector<int> devs;
    if (const char* e = std::getenv("MICS_DEVICES"))
      for (const char* p = e; *p;) {
        char* end = nullptr;
        devs.push_back(int(std::strtol(p, &end, 10)));
        p = *end ? end + 1 : end;
      }
    mics_ctx* out = nullptr;
    if (devs.size() > 1) {
      a.device = devs[0];
      check(mics_init_devices(&a, devs.data(), int(devs.size()), &out));
    } else {
      if (devs.size() == 1) a.device = devs[0];
      check(mics_init(&a, &out));
    }
    return out;
  }();
  return c;
}

// The caller's worker count (VirtualRankEngine(num_threads)) becomes the CTAs per
// SM of the call's kernels; results do not depend on it (collectives.hpp:38-41).
void use(const VirtualRankEngine& engine) { check(mics_set_parallelism(ctx(), engine.num_threads(), 0)); }

// Move the traffic libmics recorded for one call into the caller's engine log.
void collect_traffic(VirtualRankEngine& engine) {
  uint64_t n = 0;
  check(mics_traffic_size(ctx(), &n));
  std::vector<int64_t> t(3 * n + 3);
  check(mics_traffic_get(ctx(), t.data(), n));
  for (uint64_t i = 0; i < n; ++i) engine.record_traffic(int(t[3 * i]), int(t[3 * i + 1]), uint64_t(t[3 * i + 2]));
  check(mics_traffic_clear(ctx()));
}

mics_dtype to_mics(DType d) {
  switch (d) {
    case DType::i64: return MICS_I64;
    case DType::f32: return MICS_F32;
    case DType::f64: return MICS_F64;
  }
  return MICS_F32;
}

void equal_sizes(const std::vector<Bytes>& bufs, const char* what) {  // same message as the reference's check
  for (std::size_t i = 1; i < bufs.size(); ++i)
    if (bufs[i].size() != bufs[0].size())
      raise(Errc::SizeMismatch, std::string(what) + ": buffer " + std::to_string(i) + " has " +
                                    std::to_string(bufs[i].size()) + " bytes, expected " +
                                    std::to_string(bufs[0].size()));
}

struct HostViews {
  std::vector<const void*> in;
  std::vector<void*> out;
};

}  // namespace

// ---------------------------------------------------------------- topology
void ClusterSpec::validate() const {
  mics_cluster c{num_nodes, devices_per_node, intra_node_bandwidth, inter_node_bandwidth_per_node,
                 alpha_intra, alpha_inter, device_memory, device_peak_flops};
  check(mics_cluster_validate(&c));
}

GroupLayout build_group_layout(int n, int p) {
  std::vector<int> part(std::size_t(n > 0 ? n : 1)), repl(std::size_t(n > 0 ? n : 1));
  check(mics_build_group_layout(n, p, part.data(), repl.data()));
  GroupLayout l;
  l.n = n;
  l.p = p;
  for (int g = 0; g < n / p; ++g) l.partition_groups.emplace_back(part.begin() + g * p, part.begin() + (g + 1) * p);
  const int r = n / p;
  for (int j = 0; j < p; ++j) l.replication_groups.emplace_back(repl.begin() + j * r, repl.begin() + (j + 1) * r);
  return l;
}

bool partition_shape_ok(int p, int k) { return mics_partition_shape_ok(p, k) != 0; }

std::uint64_t model_state_bytes(std::uint64_t num_params, std::uint64_t bpp) {
  uint64_t out = 0;
  check(mics_model_state_bytes(num_params, bpp, &out));
  return out;
}

int min_feasible_partition(std::uint64_t states, const ClusterSpec& cl, bool node_granular, double headroom) {
  mics_cluster c{cl.num_nodes, cl.devices_per_node, cl.intra_node_bandwidth, cl.inter_node_bandwidth_per_node,
                 cl.alpha_intra, cl.alpha_inter, cl.device_memory, cl.device_peak_flops};
  int p = 0;
  check(mics_min_feasible_partition(states, &c, node_granular ? 1 : 0, headroom, &p));
  return p;
}

// ---------------------------------------------------------------- engine + traffic log
bool CollectiveGroup::spans_nodes(const ClusterSpec& cluster) const {
  for (int r : ranks)
    if (cluster.node_of(r) != cluster.node_of(ranks.front())) return true;
  return false;
}

void CollectiveGroup::validate() const {
  std::vector<char> seen;
  for (int r : ranks) {
    if (r >= int(seen.size())) seen.resize(std::size_t(r) + 1, 0);
    if (r >= 0 && seen[std::size_t(r)]++) raise(Errc::ShapeError, "collective group has duplicate ranks");
  }
}

VirtualRankEngine::VirtualRankEngine(int num_threads) : num_threads_(num_threads < 1 ? 1 : num_threads) {}

void VirtualRankEngine::parallel_for(int count, const std::function<void(int)>& fn) const {
  for (int i = 0; i < count; ++i) fn(i);  // the device does the parallel work
}

void VirtualRankEngine::record_traffic(int from, int to, std::uint64_t bytes) {
  std::lock_guard<std::mutex> lock(traffic_mu_);
  traffic_[{from, to}] += bytes;
}

std::map<std::pair<int, int>, std::uint64_t> VirtualRankEngine::traffic() const {
  std::lock_guard<std::mutex> lock(traffic_mu_);
  return traffic_;
}

std::uint64_t VirtualRankEngine::bytes_received_by(int rank) const {
  std::lock_guard<std::mutex> lock(traffic_mu_);
  std::uint64_t total = 0;
  for (const auto& kv : traffic_)
    if (kv.first.second == rank) total += kv.second;
  return total;
}

void VirtualRankEngine::clear_traffic() {
  std::lock_guard<std::mutex> lock(traffic_mu_);
  traffic_.clear();
}

// ---------------------------------------------------------------- collectives -> libmics kernels
std::vector<Bytes> all_gather(VirtualRankEngine& engine, const CollectiveGroup& group,
                              const std::vector<Bytes>& shards) {
  use(engine);
  group.validate();
  const int p = group.size();
  if (int(shards.size()) != p)
    raise(Errc::SizeMismatch, "all_gather: " + std::to_string(shards.size()) + " shards for group of " +
                                  std::to_string(p));
  equal_sizes(shards, "all_gather");
  const std::size_t chunk = shards.empty() ? 0 : shards[0].size();
  std::vector<Bytes> out(static_cast<std::size_t>(p), Bytes(std::size_t(p) * chunk));
  HostViews v;
  for (int i = 0; i < p; ++i) {
    v.in.push_back(shards[std::size_t(i)].data());
    v.out.push_back(out[std::size_t(i)].data());
  }
  check(mics_host_all_gather(ctx(), group.ranks.data(), p, v.in.data(), chunk, v.out.data()));
  collect_traffic(engine);
  return out;
}

std::vector<Bytes> reduce_scatter(VirtualRankEngine& engine, const CollectiveGroup& group,
                                  const std::vector<Bytes>& buffers, DType dtype) {
  use(engine);
  group.validate();
  const int p = group.size();
  if (int(buffers.size()) != p)
    raise(Errc::SizeMismatch, "reduce_scatter: " + std::to_string(buffers.size()) + " buffers for group of " +
                                  std::to_string(p));
  equal_sizes(buffers, "reduce_scatter");
  const std::size_t total = buffers.empty() ? 0 : buffers[0].size();
  std::vector<Bytes> out(static_cast<std::size_t>(p), Bytes(p ? total / std::size_t(p) : 0));
  HostViews v;
  for (int i = 0; i < p; ++i) {
    v.in.push_back(buffers[std::size_t(i)].data());
    v.out.push_back(out[std::size_t(i)].data());
  }
  check(mics_host_reduce_scatter(ctx(), group.ranks.data(), p, v.in.data(), total, to_mics(dtype), v.out.data()));
  collect_traffic(engine);
  return out;
}

std::vector<Bytes> all_reduce(VirtualRankEngine& engine, const CollectiveGroup& group,
                              const std::vector<Bytes>& buffers, DType dtype) {
  use(engine);
  group.validate();
  const int p = group.size();
  if (int(buffers.size()) != p)
    raise(Errc::SizeMismatch, "reduce_scatter: " + std::to_string(buffers.size()) + " buffers for group of " +
                                  std::to_string(p));
  equal_sizes(buffers, "reduce_scatter");
  const std::size_t total = buffers.empty() ? 0 : buffers[0].size();
  std::vector<Bytes> out(static_cast<std::size_t>(p), Bytes(total));
  HostViews v;
  for (int i = 0; i < p; ++i) {
    v.in.push_back(buffers[std::size_t(i)].data());
    v.out.push_back(out[std::size_t(i)].data());
  }
  check(mics_host_all_reduce(ctx(), group.ranks.data(), p, v.in.data(), total, to_mics(dtype), v.out.data()));
  collect_traffic(engine);
  return out;
}

std::vector<Bytes> hierarchical_all_gather(VirtualRankEngine& engine, const GroupLayout& layout,
                                           const ClusterSpec& cluster, const std::vector<Bytes>& shards,
                                           const HierarchicalOptions& opts) {
  use(engine);
  const int n = layout.n;
  if (cluster.total_ranks() != n)
    raise(Errc::ShapeError, "cluster has " + std::to_string(cluster.total_ranks()) + " ranks but layout expects " +
                                std::to_string(n));
  if (int(shards.size()) != n)
    raise(Errc::SizeMismatch, "hierarchical_all_gather: " + std::to_string(shards.size()) + " shards for " +
                                  std::to_string(n) + " ranks");
  equal_sizes(shards, "hierarchical_all_gather");
  const std::size_t chunk = shards[0].size();
  std::vector<Bytes> out(static_cast<std::size_t>(n), Bytes(std::size_t(layout.p) * chunk));
  HostViews v;
  for (int i = 0; i < n; ++i) {
    v.in.push_back(shards[std::size_t(i)].data());
    v.out.push_back(out[std::size_t(i)].data());
  }
  check(mics_host_hier_all_gather(ctx(), n, layout.p, cluster.devices_per_node, v.in.data(), chunk, v.out.data(),
                                  opts.corrupt_stage2 ? 1 : 0));
  collect_traffic(engine);
  return out;
}

std::vector<std::vector<Bytes>> batched_all_gather(VirtualRankEngine& engine,
                                                   const std::vector<CollectiveGroup>& groups,
                                                   const std::vector<std::vector<Bytes>>& shard_sets) {
  use(engine);
  if (groups.size() != shard_sets.size())
    raise(Errc::SizeMismatch, "batched_all_gather: " + std::to_string(groups.size()) + " groups vs " +
                                  std::to_string(shard_sets.size()) + " shard sets");
  std::vector<int> sizes, ranks;
  std::vector<uint64_t> chunks;
  std::vector<std::vector<Bytes>> out;
  HostViews v;
  for (std::size_t b = 0; b < groups.size(); ++b) {
    groups[b].validate();
    const int p = groups[b].size();
    if (int(shard_sets[b].size()) != p)
      raise(Errc::SizeMismatch, "all_gather: " + std::to_string(shard_sets[b].size()) + " shards for group of " +
                                    std::to_string(p));
    equal_sizes(shard_sets[b], "all_gather");
    const std::size_t c = shard_sets[b].empty() ? 0 : shard_sets[b][0].size();
    sizes.push_back(p);
    ranks.insert(ranks.end(), groups[b].ranks.begin(), groups[b].ranks.end());
    chunks.push_back(c);
    out.emplace_back(std::size_t(p), Bytes(std::size_t(p) * c));
  }
  for (std::size_t b = 0; b < groups.size(); ++b)
    for (std::size_t i = 0; i < out[b].size(); ++i) {
      v.in.push_back(shard_sets[b][i].data());
      v.out.push_back(out[b][i].data());
    }
  check(mics_host_batched_all_gather(ctx(), int(groups.size()), sizes.data(), ranks.data(), chunks.data(),
                                     v.in.data(), v.out.data()));
  collect_traffic(engine);
  return out;
}

std::vector<std::vector<Bytes>> batched_reduce_scatter(VirtualRankEngine& engine,
                                                       const std::vector<CollectiveGroup>& groups,
                                                       const std::vector<std::vector<Bytes>>& buffer_sets,
                                                       DType dtype) {
  use(engine);
  if (groups.size() != buffer_sets.size())
    raise(Errc::SizeMismatch, "batched_reduce_scatter: " + std::to_string(groups.size()) + " groups vs " +
                                  std::to_string(buffer_sets.size()) + " buffer sets");
  std::vector<int> sizes, ranks;
  std::vector<uint64_t> nbytes;
  std::vector<std::vector<Bytes>> out;
  HostViews v;
  for (std::size_t b = 0; b < groups.size(); ++b) {
    groups[b].validate();
    const int p = groups[b].size();
    if (int(buffer_sets[b].size()) != p)
      raise(Errc::SizeMismatch, "reduce_scatter: " + std::to_string(buffer_sets[b].size()) +
                                    " buffers for group of " + std::to_string(p));
    equal_sizes(buffer_sets[b], "reduce_scatter");
    const std::size_t total = buffer_sets[b].empty() ? 0 : buffer_sets[b][0].size();
    sizes.push_back(p);
    ranks.insert(ranks.end(), groups[b].ranks.begin(), groups[b].ranks.end());
    nbytes.push_back(total);
    out.emplace_back(std::size_t(p), Bytes(p ? total / std::size_t(p) : 0));
  }
  for (std::size_t b = 0; b < groups.size(); ++b)
    for (std::size_t i = 0; i < out[b].size(); ++i) {
      v.in.push_back(buffer_sets[b][i].data());
      v.out.push_back(out[b][i].data());
    }
  check(mics_host_batched_reduce_scatter(ctx(), int(groups.size()), sizes.data(), ranks.data(), nbytes.data(),
                                         v.in.data(), to_mics(dtype), v.out.data()));
  collect_traffic(engine);
  return out;
}

}  // namespace sdpsim
