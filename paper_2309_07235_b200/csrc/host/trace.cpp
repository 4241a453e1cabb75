// Trace files v1 (the reference format, persist.cpp:17-21, 97-222) and v2.
#include "trace.hpp"

#include <cstdio>
#include <cstdlib>
#include <sstream>

namespace tth {

namespace {

const char* const kMagicV1 = "# tiletuner-trace v1";
const char* const kMagicV2 = "# tiletuner-trace v2";
const char* const kArtifactVersion = "0.1.0";  // persist.cpp:19
const char* const kColumnsV1 = "eval_index,config,runtime_s,elapsed_s,best_so_far_s,status";
const char* const kColumnsV2 =
    "eval_index,config,runtime_s,elapsed_s,best_so_far_s,status,device,variant";

// %.17g: every finite double round-trips exactly (the reference's rule)
std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::vector<std::string> fields_of(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += ch;
    }
  }
  out.push_back(cur);
  return out;
}

double to_double(const std::string& s, int line) {
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (s.empty() || *end) throw TraceParseError("bad float '" + s + "'", line);
  return v;
}

std::uint64_t to_u64(const std::string& s, int line) {
  char* end = nullptr;
  const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
  if (s.empty() || *end || s[0] == '-') throw TraceParseError("bad integer '" + s + "'", line);
  return v;
}

long long to_i64(const std::string& s, int line) {
  char* end = nullptr;
  const long long v = std::strtoll(s.c_str(), &end, 10);
  if (s.empty() || *end) throw TraceParseError("bad integer '" + s + "'", line);
  return v;
}

bool one_of(const std::string& v, std::initializer_list<const char*> names) {
  for (const char* n : names)
    if (v == n) return true;
  return false;
}

}  // namespace

std::string format_config(const std::vector<int>& config) {
  std::string s;
  for (size_t i = 0; i < config.size(); ++i) {
    if (i) s += '|';
    s += "P" + std::to_string(i) + "=" + std::to_string(config[i]);
  }
  return s;
}

std::vector<int> parse_config(const std::string& text) {
  std::vector<int> cfg;
  if (text.empty()) return cfg;
  for (const std::string& f : fields_of(text, '|')) {
    const size_t eq = f.find('=');
    if (eq == std::string::npos) throw std::invalid_argument("bad config field '" + f + "'");
    const std::string v = f.substr(eq + 1);
    char* end = nullptr;
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end || x < 1) throw std::invalid_argument("bad config value '" + v + "'");
    cfg.push_back(static_cast<int>(x));
  }
  return cfg;
}

std::string render_trace(const Trace& trace) {
  const TraceHeader& h = trace.header;
  const bool v2 = h.version >= 2;
  std::ostringstream o;
  o << (v2 ? kMagicV2 : kMagicV1) << '\n'
    << "# version: " << kArtifactVersion << '\n'
    << "# kernel: " << h.kernel << '\n'
    << "# size: " << h.size << '\n'
    << "# tuner: " << h.tuner << '\n'
    << "# seed: " << h.seed << '\n'
    << "# max_evals: " << h.max_evals << '\n'
    << "# max_seconds: " << (h.max_seconds ? num(*h.max_seconds) : std::string("none")) << '\n'
    << "# warmups: " << h.warmups << '\n'
    << "# repetitions: " << h.repetitions << '\n'
    << "# aggregate: " << h.aggregate << '\n'
    << "# objective: " << h.objective << '\n'
    << "# created: " << h.created_unix << '\n'
    << "# total_process_s: " << num(h.total_process_s) << '\n';
  if (v2) {
    std::string devs;
    for (size_t i = 0; i < h.devices.size(); ++i) devs += (i ? "," : "") + std::to_string(h.devices[i]);
    o << "# devices: " << (devs.empty() ? std::string("none") : devs) << '\n'
      << "# batch: " << h.batch << '\n'
      << "# backend: " << (h.backend.empty() ? std::string("none") : h.backend) << '\n';
  }
  o << "# columns: " << (v2 ? kColumnsV2 : kColumnsV1) << '\n';
  for (const TraceRecord& r : trace.records) {
    o << r.eval_index << ',' << format_config(r.config) << ','
      << (r.runtime_s ? num(*r.runtime_s) : std::string("nan")) << ',' << num(r.elapsed_s) << ','
      << num(r.best_so_far_s) << ',' << (r.runtime_s ? "ok" : "fail");
    if (v2) o << ',' << r.device << ',' << (r.variant.empty() ? std::string("none") : r.variant);
    o << '\n';
  }
  return o.str();
}

Trace parse_trace(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  int no = 0;
  Trace t;
  if (!std::getline(in, line)) throw TraceParseError("missing trace header", 1);
  ++no;
  if (line == kMagicV1) {
    t.header.version = 1;
  } else if (line == kMagicV2) {
    t.header.version = 2;
  } else {
    throw TraceParseError("missing trace header", 1);
  }
  const bool v2 = t.header.version == 2;
  bool columns = false;
  while (std::getline(in, line)) {
    ++no;
    if (line.empty()) continue;
    if (line[0] == '#') {
      const size_t c = line.find(": ");
      if (c == std::string::npos || line.size() < 3) throw TraceParseError("malformed header line", no);
      const std::string key = line.substr(2, c - 2), val = line.substr(c + 2);
      TraceHeader& h = t.header;
      if (key == "version") {
        // accepted for forward compatibility
      } else if (key == "kernel") {
        if (!one_of(val, {"lu", "cholesky", "3mm"})) throw TraceParseError("unknown kernel: " + val, no);
        h.kernel = val;
      } else if (key == "size") {
        h.size = val;
      } else if (key == "tuner") {
        if (!one_of(val, {"random", "grid", "genetic", "boosted", "bayesopt"}))
          throw TraceParseError("unknown tuner: " + val, no);
        h.tuner = val;
      } else if (key == "seed") {
        h.seed = to_u64(val, no);
      } else if (key == "max_evals") {
        h.max_evals = to_u64(val, no);
      } else if (key == "max_seconds") {
        if (val == "none")
          h.max_seconds.reset();
        else
          h.max_seconds = to_double(val, no);
      } else if (key == "warmups") {
        h.warmups = static_cast<int>(to_u64(val, no));
      } else if (key == "repetitions") {
        h.repetitions = static_cast<int>(to_u64(val, no));
      } else if (key == "aggregate") {
        if (!one_of(val, {"median", "min", "mean"})) throw TraceParseError("unknown aggregate: " + val, no);
        h.aggregate = val;
      } else if (key == "objective") {
        if (!one_of(val, {"synthetic", "measured"})) throw TraceParseError("unknown objective: " + val, no);
        h.objective = val;
      } else if (key == "created") {
        h.created_unix = to_i64(val, no);
      } else if (key == "total_process_s") {
        h.total_process_s = to_double(val, no);
      } else if (v2 && key == "devices") {
        h.devices.clear();
        if (val != "none")
          for (const std::string& d : fields_of(val, ','))
            h.devices.push_back(static_cast<int>(to_u64(d, no)));
      } else if (v2 && key == "batch") {
        h.batch = static_cast<int>(to_u64(val, no));
      } else if (v2 && key == "backend") {
        h.backend = val == "none" ? std::string() : val;
      } else if (key == "columns") {
        if (val != (v2 ? kColumnsV2 : kColumnsV1)) throw TraceParseError("unexpected columns", no);
        columns = true;
      } else {
        throw TraceParseError("unknown header key '" + key + "'", no);
      }
      continue;
    }
    if (!columns) throw TraceParseError("record before columns header", no);
    const std::vector<std::string> f = fields_of(line, ',');
    if (f.size() != (v2 ? 8u : 6u))
      throw TraceParseError(v2 ? "expected 8 record fields" : "expected 6 record fields", no);
    TraceRecord r;
    r.eval_index = to_u64(f[0], no);
    try {
      r.config = parse_config(f[1]);
    } catch (const std::invalid_argument& e) {
      throw TraceParseError(e.what(), no);
    }
    if (f[5] == "ok")
      r.runtime_s = to_double(f[2], no);
    else if (f[5] != "fail")
      throw TraceParseError("bad status '" + f[5] + "'", no);
    r.elapsed_s = to_double(f[3], no);
    r.best_so_far_s = to_double(f[4], no);
    if (v2) {
      r.device = static_cast<int>(to_i64(f[6], no));
      r.variant = f[7] == "none" ? std::string() : f[7];
    }
    t.records.push_back(std::move(r));
  }
  if (!columns) throw TraceParseError("missing columns header", no == 0 ? 1 : no);
  return t;
}

bool best_of(const Trace& trace, std::vector<int>* config, double* runtime_s) {
  const TraceRecord* best = nullptr;
  for (const TraceRecord& r : trace.records)
    if (r.runtime_s && (!best || *r.runtime_s < *best->runtime_s ||
                        (*r.runtime_s == *best->runtime_s && r.eval_index < best->eval_index)))
      best = &r;
  if (!best) return false;
  if (config) *config = best->config;
  if (runtime_s) *runtime_s = *best->runtime_s;
  return true;
}

}  // namespace tth
