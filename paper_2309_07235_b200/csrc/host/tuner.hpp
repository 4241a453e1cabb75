// Host-side tuning runtime (C++17): problem registry, tile-factor search
// space, the random-forest Bayesian-optimisation tuner with a batch
// extension of the reference's ask/tell contract, and the tuning loop that
// drives the GPU objective — sequentially or as an asynchronous batched
// evaluator with one worker thread (and one tt_ctx) per GPU.
//
// Reference semantics restated here (file:line under /root/reference/proj):
//   registry        core/src/problem.cpp:25-38
//   space           core/src/space.cpp:10-124 (divisors, mixed radix, log2 encode)
//   Rng             core/include/tiletuner/rng.hpp:11-32 (mt19937_64, 53-bit doubles,
//                   128-bit multiply-shift index)
//   forest + LCB    core/src/surrogate.cpp:13-175, :209-214
//   tuner base      core/src/tuners.cpp:52-129 (ask/tell, penalty, log targets,
//                   rejection + reservoir sampling, candidate pool)
//   random / grid / bayesopt  core/src/tuners.cpp:131-139, :324-351
//   run_tuning      core/src/harness.cpp:199-265 (+ synthetic objective :166-197)
// Genetic and boosted strategies are out of scope.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <string>
#include <unordered_set>
#include <vector>

namespace tth {

enum class Kernel { lu = 0, cholesky = 1, mm3 = 2 };
enum class TunerKind { random = 0, grid = 1, genetic = 2, boosted = 3, bayesopt = 4 };

struct ProblemSize {
  Kernel kernel;
  std::string name;
  int n, l, m, o, p;
};

const std::vector<ProblemSize>& registered_sizes();
const ProblemSize* find_size(Kernel k, const std::string& name);

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  std::uint64_t next_u64() { return gen_(); }
  double next_double() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  std::uint64_t next_index(std::uint64_t n) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(gen_()) * n) >> 64);
  }

 private:
  std::mt19937_64 gen_;
};

struct Param {
  std::string name;
  int extent;
  std::vector<int> candidates;
};

struct Space {
  Kernel kernel;
  std::string size_name;
  std::vector<Param> params;
  std::uint64_t size() const;
};

std::vector<int> divisor_candidates(int n);
Space build_space(Kernel kernel, const std::string& size_name);  // throws on unknown size
std::vector<int> config_at(const Space& s, std::uint64_t flat);
bool index_of(const Space& s, const std::vector<int>& cfg, std::uint64_t* out);
std::vector<double> encode(const Space& s, const std::vector<int>& cfg);
double synthetic_objective(const Space& s, const std::vector<int>& cfg);

// ---- surrogate ----
struct Node {
  int feature = -1;
  double threshold = 0.0;
  int left = -1, right = -1;
  double value = 0.0;
};
struct Tree {
  std::vector<Node> nodes;
  double predict(const double* x) const;
};
struct Forest {
  std::vector<Tree> trees;
  int dims = 0;
};
Forest fit_forest(const std::vector<std::vector<double>>& x, const std::vector<double>& y,
                  int n_trees, int max_depth, int min_split, std::uint64_t seed);
void predict_forest(const Forest& f, const double* x, double* mean, double* std_dev);

// ---- tuners ----
class Tuner {
 public:
  Tuner(TunerKind kind, Space space, std::uint64_t seed);
  virtual ~Tuner() = default;

  // Reference contract for k = 1 (ask() then tell()); the batch extension
  // keeps a SET of pending configurations.  ask_batch(1) consumes the RNG
  // exactly like the reference's ask(), so k = 1 traces are identical.
  std::vector<std::uint64_t> ask_batch(int k);
  void tell(std::uint64_t flat, std::optional<double> runtime);

  const Space& space() const { return space_; }
  std::size_t evaluated_count() const { return hist_flat_.size(); }
  std::size_t pending_count() const { return pending_.size(); }
  TunerKind kind() const { return kind_; }

 protected:
  virtual std::vector<std::uint64_t> pick(int k) = 0;
  bool taken(std::uint64_t flat) const {
    return evaluated_.count(flat) > 0 || pending_.count(flat) > 0;
  }
  std::uint64_t sample_untaken();
  std::vector<std::uint64_t> candidate_pool();

  Space space_;
  std::uint64_t size_;
  std::uint64_t seed_;
  Rng rng_;
  std::vector<std::uint64_t> hist_flat_;
  std::vector<double> log_runtimes_;
  std::unordered_set<std::uint64_t> evaluated_;
  std::unordered_set<std::uint64_t> pending_;

 private:
  TunerKind kind_;
  double worst_ = 0.0;
};

std::unique_ptr<Tuner> make_tuner(TunerKind kind, const Space& space, std::uint64_t seed);

// ---- the tuning loop ----
struct Record {
  std::uint64_t eval_index;
  std::uint64_t flat;
  std::vector<int> config;
  std::optional<double> runtime_s;
  double elapsed_s;
  double best_so_far_s;
  int worker;
  double ask_s;   // host time spent asking for this candidate (its share of a batch ask)
  double eval_s;  // wall time of its evaluation (objective call)
};

struct TuneOptions {
  TunerKind tuner = TunerKind::bayesopt;
  Kernel kernel = Kernel::lu;
  std::string size = "large";
  std::uint64_t seed = 0;
  std::uint64_t max_evals = 100;
  std::optional<double> max_seconds;
  int workers = 1;  // batch size / number of concurrent evaluators
};

// Objective: returns runtime seconds or nullopt on a numerical failure.
// Called from worker `w` (0 <= w < workers); must be thread-safe across
// workers.  Throwing aborts the run (MeasurementError semantics).
using Objective = std::function<std::optional<double>(int worker, const std::vector<int>& cfg)>;

// Measured run: wall clock, workers evaluate concurrently, an idle worker
// gets the next candidate at once (no lock-step; with W workers the surrogate
// is fitted once per W candidates), records are appended in completion order
// (elapsed non-decreasing, best = prefix min).  An objective that throws
// (MeasurementError: device failure) retires its worker and its candidate is
// re-evaluated by another one; when no worker is left the run stops and the
// partial trace is returned with *error set (harness.cpp:252-256 flushes the
// partial trace and rethrows) — with error == nullptr it throws instead.
std::vector<Record> run_tuning(const TuneOptions& opt, const Objective& objective,
                               double* total_s, std::string* error = nullptr);

// Virtual-clock measured run (T1 / T8 harness): `workers` evaluators emulated
// on ONE real device.  Every evaluation is measured for real — the objective
// returns (runtime or nullopt, wall seconds the evaluation took) — and
// occupies its virtual evaluator for that wall time; the dispatcher's real
// host ask time is charged serially on the same clock.  Results reach the
// tuner at their virtual finish time, so the search sees exactly what a
// W-GPU run with these per-evaluation costs would see.
using VirtualObjective =
    std::function<std::pair<std::optional<double>, double>(const std::vector<int>& cfg)>;
std::vector<Record> run_tuning_virtual(const TuneOptions& opt, const VirtualObjective& objective,
                                       double* total_s, std::string* error);

// Synthetic run (harness.cpp:166-197, virtual clock): `workers` simulated
// devices, discrete-event completion order by virtual finish time.  With
// workers = 1 the trace equals the reference's run_tuning bit for bit.
std::vector<Record> run_tuning_synthetic(const TuneOptions& opt, double* total_s);

}  // namespace tth
