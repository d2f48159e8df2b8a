// TEST / TOOLING ONLY — C shim over the reference's analytical simulator
// (proj/src/{config,simulator,cost_model,units,report,topology}.cpp, compiled in place by
// oracle/Makefile `sim`).  Used by tools/b200_profile.py to feed the bandwidths measured
// on B200 back into the reference's own cost model: it runs
// `sdpsim simulate` (sdpsim_main.cpp:55-121) on a scenario file and returns the
// reference's jsonl records.
#include <cstring>
#include <string>
#include <vector>

#include "sdpsim/config.hpp"
#include "sdpsim/report.hpp"
#include "sdpsim/simulator.hpp"

using namespace sdpsim;

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* ref_sim_last_error() { return g_err.c_str(); }

// Returns 0 and writes jsonl (NUL-terminated, truncated to cap) on success.
int ref_simulate(const char* path, char* out, size_t cap) {
  try {
    ScenarioConfig cfg = load_scenario_file(path);
    validate_scenario(cfg);
    std::vector<StrategyResult> results;
    Comparison cmp;
    const bool compared = cfg.strategies.size() >= 2;
    if (compared) {
      cmp = compare_strategies(cfg.cluster, cfg.layers, cfg.strategies, cfg.sim);
      results = cmp.results;
    } else {
      results.push_back({cfg.strategies[0], simulate_iteration(cfg.cluster, cfg.layers, cfg.strategies[0], cfg.sim)});
    }
    std::vector<Json> records;
    for (std::size_t i = 0; i < results.size(); ++i) {
      const auto& r = results[i];
      Json j;
      j["scenario"] = cfg.name;
      j["strategy"] = r.config.name;
      j["total_seconds"] = r.trace.total_seconds;
      j["fwd_gather_seconds"] = r.trace.fwd_gather_seconds;
      j["bwd_gather_seconds"] = r.trace.bwd_gather_seconds;
      j["micro_sync_seconds"] = r.trace.micro_sync_seconds;
      j["boundary_sync_seconds"] = r.trace.boundary_sync_seconds;
      j["inter_node_bytes"] = r.trace.inter_node_bytes;
      j["peak_model_state_bytes_per_device"] = r.trace.peak_model_state_bytes_per_device;
      if (compared) j["throughput_ratio"] = cmp.throughput_ratio[i];
      records.push_back(std::move(j));
    }
    const std::string s = render_records(records, ReportFormat::jsonl);
    std::strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}
