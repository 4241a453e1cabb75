// tiletuner-gpu: the reference CLI's spaces | verify | tune front end
// (/root/reference/proj/tools/tiletuner.cpp:1-299) on the B200 path, with the
// device flags SURVEY.md §8(f)2 asks for:
//   tiletuner-gpu spaces <kernel> <size>
//   tiletuner-gpu verify <kernel> <size> [--samples N] [--seed S] [--device D]
//   tiletuner-gpu tune <kernel> <size> [--tuner T] [--max-evals N] [--max-seconds S]
//                 [--seed S] [--synthetic] [--reproducible] [--out PATH]
//                 [--gpus N | --devices 0,1,..] [--batch K] [--trace-format v1|v2]
// Exit codes as the reference: 0 success, 1 domain error, 2 usage error.
// verify runs the kernel on the GPU and checks the residual on the GPU
// (LU/Cholesky, kernels.cpp:326-352) or against a host-computed 3mm
// reference (mm3_reference, kernels.cpp:115-120); `tune` writes trace v2
// (device + schedule variant per record) unless --trace-format v1, which is
// the reference's format byte for byte (v1 traces of --synthetic
// --reproducible runs equal the reference CLI's output).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <fstream>
#include <iterator>
#include <iostream>
#include <set>
#include <string>
#include <vector>

#include "../../../include/tt_gpu.h"
#include "../../../include/tt_tuner.h"
#include "trace.hpp"
#include "tuner.hpp"

namespace {

constexpr std::uint64_t kInputSeed = 1;  // tiletuner.cpp:28: data seed, not the search seed

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Domain : std::runtime_error {
  using std::runtime_error::runtime_error;
};

int kernel_id(const std::string& k) {
  if (k == "lu") return TT_KERNEL_LU;
  if (k == "cholesky") return TT_KERNEL_CHOLESKY;
  if (k == "3mm" || k == "mm3") return TT_KERNEL_MM3;
  throw Usage("kernel: " + k + " not in {lu, cholesky, 3mm, mm3}");
}
const char* kernel_name(int k) { return k == TT_KERNEL_LU ? "lu" : k == TT_KERNEL_CHOLESKY ? "cholesky" : "3mm"; }

void check_size(const std::string& s) {
  if (s != "mini" && s != "small" && s != "large" && s != "extralarge")
    throw Usage("size: " + s + " not in {mini, small, large, extralarge}");
}

int tuner_id(const std::string& t) {
  const char* names[] = {"random", "grid", "genetic", "boosted", "bayesopt"};
  for (int i = 0; i < 5; ++i)
    if (t == names[i]) return i;
  throw Usage("tuner: " + t + " not in {random, grid, genetic, boosted, bayesopt}");
}

struct Args {
  std::vector<std::string> pos;
  std::vector<std::pair<std::string, std::string>> opt;
  std::set<std::string> flags;
};

Args parse_args(int argc, char** argv, int first, const std::set<std::string>& with_value,
                const std::set<std::string>& flag_names) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      std::string key = s, val;
      const size_t eq = s.find('=');
      if (eq != std::string::npos) {
        key = s.substr(0, eq);
        val = s.substr(eq + 1);
      }
      if (flag_names.count(key)) {
        a.flags.insert(key);
      } else if (with_value.count(key)) {
        if (eq == std::string::npos) {
          if (i + 1 >= argc) throw Usage(key + " needs a value");
          val = argv[++i];
        }
        a.opt.emplace_back(key, val);
      } else {
        throw Usage("unknown option " + key);
      }
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

std::string get(const Args& a, const std::string& key, const std::string& dflt) {
  std::string v = dflt;
  for (const auto& kv : a.opt)
    if (kv.first == key) v = kv.second;
  return v;
}

std::uint64_t to_u64(const std::string& key, const std::string& v) {
  char* end = nullptr;
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (v.empty() || *end || v[0] == '-') throw Usage(key + ": not a non-negative integer: " + v);
  return x;
}

double to_double(const std::string& key, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) throw Usage(key + ": not a number: " + v);
  return x;
}

// kernel + size: positional or --kernel / --size (the reference accepts both)
void problem(const Args& a, std::string* kernel, std::string* size) {
  *kernel = get(a, "--kernel", a.pos.size() > 0 ? a.pos[0] : "");
  *size = get(a, "--size", a.pos.size() > 1 ? a.pos[1] : "");
  if (kernel->empty() || size->empty()) throw Usage("kernel and size are required");
  kernel_id(*kernel);
  check_size(*size);
}

// ---- spaces (space.cpp:126-138 describe) ----
int cmd_spaces(const Args& a) {
  std::string k, s;
  problem(a, &k, &s);
  const tth::Space sp = tth::build_space(static_cast<tth::Kernel>(kernel_id(k)), s);
  for (const auto& p : sp.params) {
    std::cout << p.name << ' ' << p.extent << ' ' << p.candidates.size() << "_candidates:";
    for (size_t i = 0; i < p.candidates.size(); ++i) std::cout << (i ? "," : " ") << p.candidates[i];
    std::cout << '\n';
  }
  std::cout << "total_size: " << sp.size() << '\n';
  return 0;
}

// ---- verify ----
struct Ctx {
  tt_ctx* c = nullptr;
  explicit Ctx(int dev) {
    const int rc = tt_ctx_create(dev, &c);
    if (rc) throw Domain("no usable CUDA device " + std::to_string(dev) + " (status " + std::to_string(rc) + ")");
  }
  ~Ctx() {
    if (c) tt_ctx_destroy(c);
  }
  void check(int rc, const char* what) const {
    if (rc) throw Domain(std::string(what) + ": " + tt_last_error(c));
  }
};

// max|x - y| / max|y|
double rel_maxdiff(const std::vector<double>& x, const std::vector<double>& y) {
  double num = 0, den = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    num = std::max(num, std::fabs(x[i] - y[i]));
    den = std::max(den, std::fabs(y[i]));
  }
  return den > 0 ? num / den : num;
}

// host residuals of a (perturbed) output, for the TILETUNER_TEST_CORRUPT hook
double host_factor_residual(int kernel, const std::vector<double>& a, const std::vector<double>& f,
                            int n) {
  std::vector<double> prod(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      if (kernel == TT_KERNEL_LU) {  // L unit lower (strict part of f), U upper (with diagonal)
        for (int k = 0; k <= std::min(i, j); ++k) {
          const double l = k == i ? 1.0 : f[static_cast<size_t>(i) * n + k];
          acc += l * f[static_cast<size_t>(k) * n + j];
        }
      } else {  // L lower (with diagonal); L L^T
        for (int k = 0; k <= std::min(i, j); ++k)
          acc += f[static_cast<size_t>(i) * n + k] * f[static_cast<size_t>(j) * n + k];
      }
      prod[static_cast<size_t>(i) * n + j] = acc;
    }
  return rel_maxdiff(prod, a);
}

int cmd_verify(const Args& a) {
  std::string k, s;
  problem(a, &k, &s);
  const int kid = kernel_id(k);
  const std::uint64_t samples = to_u64("--samples", get(a, "--samples", "16"));
  const std::uint64_t seed = to_u64("--seed", get(a, "--seed", "42"));
  const int device = static_cast<int>(to_u64("--device", get(a, "--device", "0")));
  const bool corrupt = std::getenv("TILETUNER_TEST_CORRUPT") != nullptr;
  const tth::Space sp = tth::build_space(static_cast<tth::Kernel>(kid), s);
  const tth::ProblemSize* ps = tth::find_size(static_cast<tth::Kernel>(kid), s);

  // sampled configurations: tiletuner.cpp:109-121 (set of Rng::next_index draws, ascending)
  std::vector<std::vector<int>> configs;
  const std::uint64_t total = sp.size();
  if (samples >= total) {
    for (std::uint64_t i = 0; i < total; ++i) configs.push_back(tth::config_at(sp, i));
  } else {
    tth::Rng rng(seed);
    std::set<std::uint64_t> chosen;
    while (chosen.size() < samples) chosen.insert(rng.next_index(total));
    for (std::uint64_t f : chosen) configs.push_back(tth::config_at(sp, f));
  }

  Ctx ctx(device);
  ctx.check(tt_setup_seeded(ctx.c, kid, ps->n, ps->l, ps->m, ps->o, ps->p, kInputSeed), "setup");
  std::vector<double> ref;  // 3mm: mm3_reference on the host (ascending-k dot products)
  std::vector<double> in_a;
  const int n = ps->n;
  if (kid == TT_KERNEL_MM3) {
    const int l = ps->l, m = ps->m, o = ps->o, p = ps->p;
    std::vector<double> A(static_cast<size_t>(n) * l), B(static_cast<size_t>(l) * m),
        C(static_cast<size_t>(m) * o), D(static_cast<size_t>(o) * p);
    ctx.check(tt_get_input(ctx.c, A.data(), B.data(), C.data(), D.data()), "inputs");
    auto mm = [](const std::vector<double>& x, const std::vector<double>& y, int r, int kk, int c) {
      std::vector<double> out(static_cast<size_t>(r) * c);
      for (int i = 0; i < r; ++i)
        for (int j = 0; j < c; ++j) {
          double acc = 0.0;
          for (int q = 0; q < kk; ++q) acc += x[static_cast<size_t>(i) * kk + q] * y[static_cast<size_t>(q) * c + j];
          out[static_cast<size_t>(i) * c + j] = acc;
        }
      return out;
    };
    ref = mm(mm(A, B, n, l, m), mm(C, D, m, o, p), n, m, p);
  } else if (corrupt) {
    in_a.resize(static_cast<size_t>(n) * n);
    ctx.check(tt_get_input(ctx.c, in_a.data(), nullptr, nullptr, nullptr), "inputs");
  }

  bool all = true;
  for (const auto& cfg : configs) {
    int fail = -1;
    double res = 0.0;
    const size_t out_n = kid == TT_KERNEL_MM3 ? static_cast<size_t>(n) * ps->p : static_cast<size_t>(n) * n;
    if (corrupt) {
      std::vector<double> out(out_n);
      ctx.check(tt_run(ctx.c, cfg.data(), static_cast<int>(cfg.size()), out.data(), &fail), "run");
      out[0] += 1.0;
      if (kid == TT_KERNEL_MM3) {
        res = rel_maxdiff(out, ref);
      } else {
        if (kid == TT_KERNEL_CHOLESKY)  // lower_of: the upper triangle keeps A's values
          for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) out[static_cast<size_t>(i) * n + j] = 0.0;
        res = host_factor_residual(kid, in_a, out, n);
      }
    } else {
      ctx.check(tt_run(ctx.c, cfg.data(), static_cast<int>(cfg.size()), nullptr, &fail), "run");
      ctx.check(tt_residual(ctx.c, kid == TT_KERNEL_MM3 ? ref.data() : nullptr, &res), "residual");
    }
    const bool pass = res <= 1e-10;
    all &= pass;
    char b[32];
    std::snprintf(b, sizeof b, "%.3e", res);
    std::cout << k << ' ' << s << ' ' << tth::format_config(cfg) << ' ' << b << ' '
              << (pass ? "PASS" : "FAIL") << '\n';
  }
  return all ? 0 : 1;
}

// ---- tune ----
std::string variant_of(int kid, const std::vector<int>& cfg, int n) {
  if (kid == TT_KERNEL_MM3) return "dgemm";
  const char* forced = std::getenv("TT_FACTOR_SCHEDULE");
  if (forced && std::string(forced) == "graph") return "graph";
  return tt_dag_urgent(kid, n, cfg[0], cfg[1]) >= 0 ? "dag" : "graph";
}

int cmd_tune(const Args& a) {
  std::string k, s;
  problem(a, &k, &s);
  const int kid = kernel_id(k);
  const std::string tuner = get(a, "--tuner", "bayesopt");
  const int tid = tuner_id(tuner);
  const std::uint64_t max_evals = to_u64("--max-evals", get(a, "--max-evals", "100"));
  const double max_seconds = to_double("--max-seconds", get(a, "--max-seconds", "0"));
  const std::uint64_t seed = to_u64("--seed", get(a, "--seed", "42"));
  const bool synthetic = a.flags.count("--synthetic") > 0;
  const std::string fmt = get(a, "--trace-format", "v2");
  if (fmt != "v1" && fmt != "v2") throw Usage("--trace-format: v1 or v2");
  std::vector<int> devices;
  const std::string dl = get(a, "--devices", "");
  if (!dl.empty()) {
    size_t pos = 0;
    while (pos <= dl.size()) {
      const size_t c = dl.find(',', pos);
      devices.push_back(static_cast<int>(to_u64("--devices", dl.substr(pos, c - pos))));
      if (c == std::string::npos) break;
      pos = c + 1;
    }
  } else {
    const int g = static_cast<int>(to_u64("--gpus", get(a, "--gpus", "1")));
    if (g < 1) throw Usage("--gpus must be >= 1");
    for (int i = 0; i < g; ++i) devices.push_back(i);
  }
  const int batch = static_cast<int>(to_u64("--batch", get(a, "--batch", synthetic ? "1" : std::to_string(devices.size()))));
  if (batch < 1) throw Usage("--batch must be >= 1");
  if (max_evals < 1) throw Domain("run_tuning: max_evals must be >= 1");
  if (tid == 2 || tid == 3) throw Domain("tuner " + tuner + " is not provided by the B200 runtime");
  const std::string out = get(a, "--out", std::string(kernel_name(kid)) + "_" + s + "_" + tuner + ".trace");

  // measurement protocol: MeasureProtocol{} + TILETUNER_REPS (harness.cpp:42-51)
  int warmups = 1, reps = 3;
  if (const char* r = std::getenv("TILETUNER_REPS")) {
    char* end = nullptr;
    const long v = std::strtol(r, &end, 10);
    if (end != r && *end == '\0' && v > 0) reps = static_cast<int>(v);
  }
  const tth::ProblemSize* ps = tth::find_size(static_cast<tth::Kernel>(kid), s);
  std::vector<tt_record> rec(max_evals);
  int got = 0;
  double total = 0.0;
  const std::int64_t created = static_cast<std::int64_t>(std::time(nullptr));
  std::string failure;
  if (synthetic) {
    const int rc = tt_tune_synthetic(tid, kid, s.c_str(), seed, static_cast<int>(max_evals), max_seconds,
                                     batch, rec.data(), static_cast<int>(rec.size()), &got, &total);
    if (rc) throw Domain("synthetic tuning failed (status " + std::to_string(rc) + ")");
  } else {
    char err[512] = {0};
    if (batch != static_cast<int>(devices.size())) {  // --batch K: K evaluators over the devices
      // K > devices puts several timed evaluators on one GPU: their event
      // windows overlap (the persistent kernel fills the GPU), so the runtimes
      // the tuner learns are contended — a functional-test mode, said so here
      if (batch > static_cast<int>(devices.size()))
        std::fprintf(stderr,
                     "warning: --batch %d > %zu device(s): evaluators share a GPU and time each "
                     "other's kernels (functional-test mode, not a tuning measurement)\n",
                     batch, devices.size());
      std::vector<int> d;
      for (int i = 0; i < batch; ++i) d.push_back(devices[i % devices.size()]);
      devices = d;
    }
    const int rc = tt_tune_measured(tid, kid, s.c_str(), seed, kInputSeed, static_cast<int>(max_evals),
                                    max_seconds, devices.data(), static_cast<int>(devices.size()), warmups,
                                    reps, 0, 1, rec.data(), static_cast<int>(rec.size()), &got, &total, err,
                                    sizeof err);
    // MeasurementError: the partial trace is still written (harness.cpp:252-256
    // flushes it before rethrowing); the error is reported after the flush
    if (rc && !(rc == TT_EDEVICE && got > 0)) throw Domain(std::string("measured tuning failed: ") + err);
    if (rc) failure = std::string("measured tuning failed (partial trace flushed): ") + err;
  }

  tth::Trace tr;
  tth::TraceHeader& h = tr.header;
  h.version = fmt == "v1" ? 1 : 2;
  h.kernel = kernel_name(kid);
  h.size = s;
  h.tuner = tuner;
  h.seed = seed;
  h.max_evals = max_evals;
  if (max_seconds > 0) h.max_seconds = max_seconds;
  h.warmups = warmups;
  h.repetitions = reps;
  h.aggregate = "median";
  h.objective = synthetic ? "synthetic" : "measured";
  h.created_unix = a.flags.count("--reproducible") ? 0 : created;
  h.total_process_s = total;
  if (!synthetic) h.devices = devices;
  h.batch = synthetic ? batch : static_cast<int>(devices.size());
  h.backend = synthetic ? "none" : std::string("b200-sm_100a");
  for (int i = 0; i < got; ++i) {
    tth::TraceRecord r;
    r.eval_index = rec[i].eval_index;
    r.config.assign(rec[i].config, rec[i].config + rec[i].nconfig);
    if (!rec[i].failed) r.runtime_s = rec[i].runtime_s;
    r.elapsed_s = rec[i].elapsed_s;
    r.best_so_far_s = rec[i].best_so_far_s;
    r.device = synthetic ? -1 : devices[rec[i].worker];
    r.variant = synthetic ? "synthetic" : variant_of(kid, r.config, ps->n);
    tr.records.push_back(std::move(r));
  }
  {
    std::ofstream f(out, std::ios::binary);
    if (!f) throw Domain("cannot open for writing: " + out);
    f << tth::render_trace(tr);
    if (!f.flush()) throw Domain("write failed: " + out);
  }
  if (!failure.empty()) throw Domain(failure);
  // report_best (tiletuner.cpp:139-151)
  std::cout << "trace: " << out << '\n' << "evals: " << tr.records.size() << '\n';
  std::vector<int> best;
  double rt = 0;
  if (!tth::best_of(tr, &best, &rt)) throw Domain("best_of: trace holds no successful evaluation");
  char b[40];
  std::cout << "best_config: " << tth::format_config(best) << '\n';
  std::snprintf(b, sizeof b, "%.6g", rt);
  std::cout << "best_runtime_s: " << b << '\n';
  std::snprintf(b, sizeof b, "%.6g", total);
  std::cout << "total_process_s: " << b << '\n';
  return 0;
}

// ---- show: read a trace (v1 or v2) and report its best record ----
int cmd_show(const Args& a) {
  if (a.pos.size() != 1) throw Usage("show needs one trace path");
  std::ifstream f(a.pos[0], std::ios::binary);
  if (!f) throw Domain("cannot open for reading: " + a.pos[0]);
  const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  const tth::Trace tr = tth::parse_trace(text);
  std::vector<int> best;
  double rt = 0;
  std::cout << "version: v" << tr.header.version << '\n'
            << "kernel: " << tr.header.kernel << '\n'
            << "size: " << tr.header.size << '\n'
            << "evals: " << tr.records.size() << '\n';
  if (tth::best_of(tr, &best, &rt)) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", rt);
    std::cout << "best_config: " << tth::format_config(best) << '\n' << "best_runtime_s: " << b << '\n';
  }
  std::set<int> devs;
  for (const auto& r : tr.records)
    if (r.device >= 0) devs.insert(r.device);
  std::cout << "devices_used:";
  for (int d : devs) std::cout << ' ' << d;
  std::cout << '\n';
  // a v2 trace re-rendered as v1 (what the reference's parser reads)
  if (a.flags.count("--as-v1")) {
    tth::Trace v1 = tr;
    v1.header.version = 1;
    std::cout << tth::render_trace(v1);
  }
  return 0;
}

void usage(std::ostream& o) {
  o << "usage: tiletuner-gpu {spaces|verify|tune} <kernel> <size> [options]\n"
       "       tiletuner-gpu show <trace> [--as-v1]\n"
       "  kernel: lu | cholesky | 3mm | mm3     size: mini | small | large | extralarge\n"
       "  verify: --samples N --seed S --device D\n"
       "  tune:   --tuner {random,grid,bayesopt} --max-evals N --max-seconds S --seed S\n"
       "          --synthetic --reproducible --out PATH --gpus N | --devices 0,1 --batch K\n"
       "          --trace-format {v1,v2}\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return 2;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage(std::cout);
    return 0;
  }
  try {
    if (cmd == "spaces") return cmd_spaces(parse_args(argc, argv, 2, {"--kernel", "--size"}, {}));
    if (cmd == "verify")
      return cmd_verify(parse_args(argc, argv, 2, {"--kernel", "--size", "--samples", "--seed", "--device"}, {}));
    if (cmd == "tune")
      return cmd_tune(parse_args(argc, argv, 2,
                                 {"--kernel", "--size", "--tuner", "--max-evals", "--max-seconds", "--seed",
                                  "--out", "--gpus", "--devices", "--batch", "--trace-format"},
                                 {"--synthetic", "--reproducible"}));
    if (cmd == "show") return cmd_show(parse_args(argc, argv, 2, {}, {"--as-v1"}));
    throw Usage("unknown command " + cmd);
  } catch (const tth::TraceParseError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << '\n';
    usage(std::cerr);
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
