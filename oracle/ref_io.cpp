// TEST INFRASTRUCTURE ONLY: the reference's report writer (core/src/io.cpp:
// write_report, config_echo, parse_config) behind a flat C entry point, so
// tests/test_report.py can compare the product's report files with the
// reference's own output for the same report and config.
#include <cstdint>
#include <exception>
#include <string>

#include "smalign/io.hpp"
#include "smalign/solver.hpp"

using namespace smalign;

extern "C" {

// config_path: a key = value config file (parse_config); vals: best_value,
// global_lower, gap, r[3], t[3], wall_time; stats: branches_expanded,
// sma_invocations, bound_evaluations; trace: n x 8 rows (wave, evals,
// best_upper, global_lower, queue_size, unexplored, pruned, resolved).
// Returns 0 on success.
int ref_write_report(const char* config_path, const double* vals, int status,
                     const unsigned long long* stats, const double* trace, long n_trace,
                     const char* epsilon_interpretation, const char* out_path, int csv) {
  try {
    const RunConfig cfg = parse_config(config_path);
    SolverReport r;
    r.best_value = vals[0];
    r.global_lower = vals[1];
    r.gap = vals[2];
    for (int k = 0; k < 3; ++k) {
      r.best_pose.r[k] = vals[3 + k];
      r.best_pose.t[k] = vals[6 + k];
    }
    r.stats.wall_time_seconds = vals[9];
    r.status = status == 0 ? SolverStatus::epsilon_optimal
               : status == 1 ? SolverStatus::time_limit
                             : SolverStatus::queue_exhausted;
    r.epsilon_interpretation = epsilon_interpretation;
    r.stats.branches_expanded = stats[0];
    r.stats.sma_invocations = stats[1];
    r.stats.bound_evaluations = stats[2];
    for (long i = 0; i < n_trace; ++i) {
      const double* t = trace + 8 * i;
      TraceEntry e;
      e.wave = static_cast<std::uint64_t>(t[0]);
      e.bound_evaluations = static_cast<std::uint64_t>(t[1]);
      e.best_upper = t[2];
      e.global_lower = t[3];
      e.queue_size = static_cast<std::size_t>(t[4]);
      e.unexplored_volume_fraction = t[5];
      e.pruned_volume_fraction = t[6];
      e.resolved_volume_fraction = t[7];
      r.trace.push_back(e);
    }
    write_report(r, cfg, out_path, csv ? ReportFormat::trace_csv : ReportFormat::json);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"
