// Tuning-trace files: the reference's v1 text format (persist.cpp:17-21,
// 97-222, rendered byte for byte) and v2, which adds what a multi-GPU run
// needs: the device that measured each record, the schedule variant that ran,
// and the evaluator layout (devices, batch).  The reader accepts both; v1 files
// written here parse with the reference's own parse_trace.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace tth {

struct TraceParseError : std::runtime_error {
  TraceParseError(const std::string& what, int line)
      : std::runtime_error("line " + std::to_string(line) + ": " + what), line(line) {}
  int line;
};

struct TraceRecord {
  std::uint64_t eval_index = 0;
  std::vector<int> config;
  std::optional<double> runtime_s;  // nullopt: failed evaluation
  double elapsed_s = 0.0;
  double best_so_far_s = 0.0;
  int device = -1;                  // v2: device that measured it (-1: none / v1)
  std::string variant;              // v2: schedule that ran ("dag", "graph", "dgemm", "synthetic")
};

struct TraceHeader {
  int version = 2;
  std::string kernel = "lu";        // "lu" | "cholesky" | "3mm"
  std::string size = "large";
  std::string tuner = "bayesopt";
  std::uint64_t seed = 0;
  std::uint64_t max_evals = 0;
  std::optional<double> max_seconds;
  int warmups = 1;
  int repetitions = 3;
  std::string aggregate = "median";
  std::string objective = "measured";  // "synthetic" | "measured"
  std::int64_t created_unix = 0;
  double total_process_s = 0.0;
  std::vector<int> devices;         // v2
  int batch = 1;                    // v2: concurrent evaluators
  std::string backend;              // v2: e.g. "b200-sm_100a"
};

struct Trace {
  TraceHeader header;
  std::vector<TraceRecord> records;
};

std::string format_config(const std::vector<int>& config);          // "P0=v0|P1=v1|..."
std::vector<int> parse_config(const std::string& text);             // throws std::invalid_argument
std::string render_trace(const Trace& trace);                       // header.version selects v1 / v2
Trace parse_trace(const std::string& text);                         // v1 or v2; throws TraceParseError
// Best successful record (earliest eval_index on ties); false if none.
bool best_of(const Trace& trace, std::vector<int>* config, double* runtime_s);

}  // namespace tth
