// Host-side tuning runtime — see tuner.hpp for the reference map.
#include "tuner.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <thread>

namespace tth {

// ------------------------------------------------------------ registry/space

const std::vector<ProblemSize>& registered_sizes() {
  static const std::vector<ProblemSize> reg = [] {
    std::vector<ProblemSize> v;
    const struct { const char* name; int n; } sq[] = {
        {"mini", 64}, {"small", 400}, {"large", 2000}, {"extralarge", 4000}};
    for (Kernel k : {Kernel::lu, Kernel::cholesky})
      for (const auto& s : sq) v.push_back({k, s.name, s.n, 0, 0, 0, 0});
    v.push_back({Kernel::mm3, "mini", 16, 18, 20, 22, 24});
    v.push_back({Kernel::mm3, "small", 80, 90, 100, 110, 120});
    v.push_back({Kernel::mm3, "large", 800, 900, 1000, 1100, 1200});
    v.push_back({Kernel::mm3, "extralarge", 1600, 1800, 2000, 2200, 2400});
    return v;
  }();
  return reg;
}

const ProblemSize* find_size(Kernel k, const std::string& name) {
  for (const auto& s : registered_sizes())
    if (s.kernel == k && s.name == name) return &s;
  return nullptr;
}

std::uint64_t Space::size() const {
  std::uint64_t t = 1;
  for (const auto& p : params) t *= p.candidates.size();
  return t;
}

std::vector<int> divisor_candidates(int n) {
  if (n < 1) throw std::invalid_argument("divisor_candidates: n must be >= 1");
  std::vector<int> out;
  for (int d = 1; d <= n; ++d)
    if (n % d == 0) out.push_back(d);  // ascending, same list as space.cpp:10-20
  return out;
}

Space build_space(Kernel kernel, const std::string& size_name) {
  const ProblemSize* s = find_size(kernel, size_name);
  if (!s) throw std::out_of_range("unregistered problem size: " + size_name);
  Space sp{kernel, size_name, {}};
  // axis extents in schedule order (space.cpp:36): E rows/cols, F rows/cols, G rows/cols
  std::vector<int> ext = kernel == Kernel::mm3
                             ? std::vector<int>{s->n, s->m, s->m, s->p, s->n, s->p}
                             : std::vector<int>{s->n, s->n};
  for (std::size_t i = 0; i < ext.size(); ++i)
    sp.params.push_back({"P" + std::to_string(i), ext[i], divisor_candidates(ext[i])});
  return sp;
}

std::vector<int> config_at(const Space& s, std::uint64_t flat) {
  if (flat >= s.size()) throw std::invalid_argument("config_at: flat index out of range");
  std::vector<int> cfg(s.params.size());
  for (std::size_t i = s.params.size(); i-- > 0;) {  // last parameter fastest
    const auto& c = s.params[i].candidates;
    cfg[i] = c[flat % c.size()];
    flat /= c.size();
  }
  return cfg;
}

bool index_of(const Space& s, const std::vector<int>& cfg, std::uint64_t* out) {
  if (cfg.size() != s.params.size()) return false;
  std::uint64_t idx = 0;
  for (std::size_t i = 0; i < cfg.size(); ++i) {
    const auto& c = s.params[i].candidates;
    auto it = std::lower_bound(c.begin(), c.end(), cfg[i]);
    if (it == c.end() || *it != cfg[i]) return false;
    idx = idx * c.size() + static_cast<std::uint64_t>(it - c.begin());
  }
  *out = idx;
  return true;
}

std::vector<double> encode(const Space& s, const std::vector<int>& cfg) {
  std::uint64_t tmp;
  if (!index_of(s, cfg, &tmp)) throw std::invalid_argument("encode: configuration not in space");
  std::vector<double> f(cfg.size());
  for (std::size_t i = 0; i < cfg.size(); ++i) f[i] = std::log2(static_cast<double>(cfg[i]));
  return f;
}

// harness.cpp:166-197: t = 1 + sum (log2 c - log2 c*)^2, c* = candidate
// nearest sqrt(extent), ties to the smaller.
double synthetic_objective(const Space& s, const std::vector<int>& cfg) {
  double t = 1.0;
  for (std::size_t i = 0; i < s.params.size(); ++i) {
    const auto& p = s.params[i];
    const double target = std::sqrt(static_cast<double>(p.extent));
    int best = p.candidates.front();
    double bd = std::abs(static_cast<double>(best) - target);
    for (int c : p.candidates) {
      const double d = std::abs(static_cast<double>(c) - target);
      if (d < bd) {
        best = c;
        bd = d;
      }
    }
    const double d = std::log2(static_cast<double>(cfg[i])) - std::log2(static_cast<double>(best));
    t += d * d;
  }
  return t;
}

// ------------------------------------------------------------------- forest

double Tree::predict(const double* x) const {
  int i = 0;
  while (nodes[i].feature >= 0) i = x[nodes[i].feature] <= nodes[i].threshold ? nodes[i].left
                                                                              : nodes[i].right;
  return nodes[i].value;
}

namespace {

using Mat = std::vector<std::vector<double>>;

struct Split {
  int feature = -1;
  double threshold = 0.0;
  double sse = std::numeric_limits<double>::infinity();
};

// Variance-reduction split (surrogate.cpp:39-75): per feature, rows sorted by
// (value, index); prefix sums in that order; midpoint thresholds between
// distinct consecutive values; first strictly-best candidate wins.
Split best_split(const Mat& x, const std::vector<double>& y, const std::vector<int>& idx,
                 int dims) {
  Split best;
  const int n = static_cast<int>(idx.size());
  std::vector<int> ord(idx);
  for (int f = 0; f < dims; ++f) {
    std::sort(ord.begin(), ord.end(), [&](int a, int b) {
      return x[a][f] != x[b][f] ? x[a][f] < x[b][f] : a < b;
    });
    double tot = 0.0, tot2 = 0.0;
    for (int i : ord) {
      tot += y[i];
      tot2 += y[i] * y[i];
    }
    double ls = 0.0, ls2 = 0.0;
    for (int r = 0; r + 1 < n; ++r) {
      const int i = ord[r];
      ls += y[i];
      ls2 += y[i] * y[i];
      if (x[i][f] == x[ord[r + 1]][f]) continue;
      const int nl = r + 1, nr = n - nl;
      const double rs = tot - ls, rs2 = tot2 - ls2;
      const double sse = (ls2 - ls * ls / nl) + (rs2 - rs * rs / nr);
      if (sse < best.sse) {
        best = {f, 0.5 * (x[i][f] + x[ord[r + 1]][f]), sse};
      }
    }
  }
  return best;
}

int grow(Tree& t, const Mat& x, const std::vector<double>& y, std::vector<int> idx, int depth,
         int max_depth, int min_split, int dims) {
  const int id = static_cast<int>(t.nodes.size());
  t.nodes.emplace_back();
  double s = 0.0;
  for (int i : idx) s += y[i];
  t.nodes[id].value = s / static_cast<double>(idx.size());
  if (depth >= max_depth || static_cast<int>(idx.size()) < min_split) return id;
  const Split sp = best_split(x, y, idx, dims);
  if (sp.feature < 0) return id;
  std::vector<int> li, ri;
  for (int i : idx) (x[i][sp.feature] <= sp.threshold ? li : ri).push_back(i);
  if (li.empty() || ri.empty()) return id;
  idx.clear();
  idx.shrink_to_fit();
  const int l = grow(t, x, y, std::move(li), depth + 1, max_depth, min_split, dims);
  const int r = grow(t, x, y, std::move(ri), depth + 1, max_depth, min_split, dims);
  t.nodes[id].feature = sp.feature;
  t.nodes[id].threshold = sp.threshold;
  t.nodes[id].left = l;
  t.nodes[id].right = r;
  return id;
}

}  // namespace

// Runs body(i) for i in [0, n) on up to `threads` host threads (static
// round-robin assignment; the result of each i does not depend on the order).
template <class F>
void parallel_for(int n, int threads, F&& body) {
  threads = std::max(1, std::min(threads, n));
  if (threads == 1) {
    for (int i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads - 1);
  for (int w = 1; w < threads; ++w)
    pool.emplace_back([&, w] {
      for (int i = w; i < n; i += threads) body(i);
    });
  for (int i = 0; i < n; i += threads) body(i);
  for (auto& th : pool) th.join();
}

int host_threads() {
  static const int n = [] {
    const unsigned hw = std::thread::hardware_concurrency();
    return static_cast<int>(std::max(1u, std::min(hw, 16u)));
  }();
  return n;
}

// surrogate.cpp:140-160.  The bootstrap samples of every tree are drawn first,
// in tree order, from the one seeded stream — exactly the draws of the
// sequential fit — and the trees are then grown in parallel (growing uses no
// randomness), so the forest is the same for any thread count.
Forest fit_forest(const Mat& x, const std::vector<double>& y, int n_trees, int max_depth,
                  int min_split, std::uint64_t seed) {
  if (x.empty() || x.size() != y.size()) throw std::invalid_argument("fit_forest: bad data");
  Forest f;
  f.dims = static_cast<int>(x.front().size());
  Rng rng(seed);
  const int n = static_cast<int>(x.size());
  std::vector<std::vector<int>> boot(n_trees, std::vector<int>(n));
  for (auto& idx : boot)
    for (int& i : idx) i = static_cast<int>(rng.next_index(n));  // bootstrap
  f.trees.resize(n_trees);
  parallel_for(n_trees, host_threads(), [&](int t) {
    grow(f.trees[t], x, y, std::move(boot[t]), 0, max_depth, min_split, f.dims);
  });
  return f;
}

void predict_forest(const Forest& f, const double* x, double* mean, double* sd) {
  std::vector<double> p;
  p.reserve(f.trees.size());
  for (const auto& t : f.trees) p.push_back(t.predict(x));
  bool same = true;
  double s = 0.0;
  for (double v : p) {
    same &= v == p.front();
    s += v;
  }
  if (same) {
    *mean = p.front();
    *sd = 0.0;
    return;
  }
  const double n = static_cast<double>(p.size());
  const double m = s / n;
  double var = 0.0;
  for (double v : p) var += (v - m) * (v - m);
  *mean = m;
  *sd = std::sqrt(var / n);
}

// ------------------------------------------------------------------- tuners

Tuner::Tuner(TunerKind kind, Space space, std::uint64_t seed)
    : space_(std::move(space)), size_(space_.size()), seed_(seed), rng_(seed), kind_(kind) {}

std::vector<std::uint64_t> Tuner::ask_batch(int k) {
  if (k < 1) throw std::invalid_argument("ask_batch: k must be >= 1");
  const std::uint64_t left = size_ - evaluated_.size() - pending_.size();
  if (left == 0) return {};  // SpaceExhausted
  std::vector<std::uint64_t> got = pick(static_cast<int>(std::min<std::uint64_t>(k, left)));
  for (auto f : got) pending_.insert(f);
  return got;
}

void Tuner::tell(std::uint64_t flat, std::optional<double> runtime) {
  if (!pending_.erase(flat)) throw std::invalid_argument("tell(): configuration was not asked");
  double eff;
  if (runtime) {
    worst_ = std::max(worst_, *runtime);
    eff = *runtime;
  } else {
    eff = worst_ > 0.0 ? 10.0 * worst_ : 1e6;  // tuners.cpp:66-74
  }
  hist_flat_.push_back(flat);
  evaluated_.insert(flat);
  log_runtimes_.push_back(std::log(std::max(eff, 1e-12)));
}

std::uint64_t Tuner::sample_untaken() {
  for (int tries = 0; tries < 1000; ++tries) {
    const std::uint64_t f = rng_.next_index(size_);
    if (!taken(f)) return f;
  }
  std::uint64_t chosen = size_, seen = 0;  // reservoir pass (tuners.cpp:88-98)
  for (std::uint64_t i = 0; i < size_; ++i) {
    if (taken(i)) continue;
    ++seen;
    if (rng_.next_index(seen) == 0) chosen = i;
  }
  return chosen;
}

std::vector<std::uint64_t> Tuner::candidate_pool() {
  std::vector<std::uint64_t> pool;
  if (size_ <= 4096) {
    for (std::uint64_t i = 0; i < size_; ++i)
      if (!taken(i)) pool.push_back(i);
    return pool;
  }
  std::unordered_set<std::uint64_t> drawn;
  for (int t = 0; t < 20 * 2048 && static_cast<int>(drawn.size()) < 2048; ++t) {
    const std::uint64_t f = rng_.next_index(size_);
    if (!taken(f)) drawn.insert(f);
  }
  pool.assign(drawn.begin(), drawn.end());
  std::sort(pool.begin(), pool.end());
  return pool;
}

namespace {

class RandomTuner final : public Tuner {
 public:
  using Tuner::Tuner;

 protected:
  std::vector<std::uint64_t> pick(int k) override {
    std::vector<std::uint64_t> out;
    for (int i = 0; i < k; ++i) {
      out.push_back(sample_untaken());
      pending_.insert(out.back());  // visible to the next draw of this batch
    }
    for (auto f : out) pending_.erase(f);
    return out;
  }
};

class GridTuner final : public Tuner {
 public:
  using Tuner::Tuner;

 protected:
  std::vector<std::uint64_t> pick(int k) override {
    std::vector<std::uint64_t> out;
    while (static_cast<int>(out.size()) < k && cursor_ < size_) out.push_back(cursor_++);
    return out;
  }

 private:
  std::uint64_t cursor_ = 0;
};

class BayesOptTuner final : public Tuner {
 public:
  BayesOptTuner(Space s, std::uint64_t seed)
      : Tuner(TunerKind::bayesopt, std::move(s), seed),
        init_(std::max(4, 2 * static_cast<int>(space_.params.size()))) {}

 protected:
  // tuners.cpp:331-351 for k = 1.  k > 1: one forest fit and one pool,
  // the k best LCB scores (ties to the lower flat index).
  // Warm-up: random untaken configs until init_ configs have RESULTS (the
  // reference's history_.size() < init_size_, tuners.cpp:333-335); with
  // several evaluators in flight that can be more than init_ random asks.
  // Never returns fewer than k unless the space is exhausted.
  std::vector<std::uint64_t> pick(int k) override {
    std::vector<std::uint64_t> out;
    if (hist_flat_.size() < static_cast<std::size_t>(init_)) {
      while (static_cast<int>(out.size()) < k) {
        const std::uint64_t f = sample_untaken();
        if (f >= size_) break;  // exhausted
        out.push_back(f);
        pending_.insert(f);
      }
      for (auto f : out) pending_.erase(f);
      return out;
    }
    const int need = k;
    for (auto f : out) pending_.insert(f);
    std::vector<std::uint64_t> pool = candidate_pool();
    for (auto f : out) pending_.erase(f);
    if (pool.empty()) return out;
    std::vector<std::vector<double>> X;
    X.reserve(hist_flat_.size());
    for (auto f : hist_flat_) X.push_back(encode(space_, config_at(space_, f)));
    const Forest model = fit_forest(X, log_runtimes_, 25, 12, 2, seed_);
    std::vector<std::pair<double, std::uint64_t>> scored(pool.size());
    std::vector<std::pair<double, double>> pred(pool.size());  // (mean, sd) per candidate
    const int np = static_cast<int>(pool.size());
    const int chunks = std::min(host_threads(), std::max(1, np / 256));
    parallel_for(chunks, chunks, [&](int c) {
      for (int i = c; i < np; i += chunks) {
        const auto e = encode(space_, config_at(space_, pool[i]));
        double m, sd;
        predict_forest(model, e.data(), &m, &sd);
        scored[i] = {m - 1.96 * sd, pool[i]};  // lcb, kappa = 1.96 (tuners.hpp:172-176)
        pred[i] = {m, sd};
      }
    });
    if (need == 1) {  // first strict minimum over the ascending pool
      auto best = scored.front();
      for (const auto& p : scored)
        if (p.first < best.first) best = p;
      out.push_back(best.second);
    } else {
      // k best LCB scores, one per model cell first: candidates whose (mean,
      // sd) equals an already chosen one's fall in the same leaf of every
      // tree — the forest cannot tell them apart, so a batch of them would
      // spend k evaluations on one prediction.  Cells are skipped until each
      // chosen candidate is from a distinct cell, then the batch is filled in
      // score order.
      std::vector<int> order(np);
      for (int i = 0; i < np; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(),
                       [&](int a, int b) { return scored[a].first < scored[b].first; });
      std::vector<std::pair<double, double>> cells;
      std::vector<int> skipped;
      for (int i : order) {
        if (static_cast<int>(out.size()) == need) break;
        if (std::find(cells.begin(), cells.end(), pred[i]) != cells.end()) {
          skipped.push_back(i);
          continue;
        }
        cells.push_back(pred[i]);
        out.push_back(scored[i].second);
      }
      for (int i : skipped) {
        if (static_cast<int>(out.size()) == need) break;
        out.push_back(scored[i].second);
      }
    }
    return out;
  }

 private:
  int init_;
};

}  // namespace

std::unique_ptr<Tuner> make_tuner(TunerKind kind, const Space& space, std::uint64_t seed) {
  switch (kind) {
    case TunerKind::random: return std::make_unique<RandomTuner>(TunerKind::random, space, seed);
    case TunerKind::grid: return std::make_unique<GridTuner>(TunerKind::grid, space, seed);
    case TunerKind::bayesopt: return std::make_unique<BayesOptTuner>(space, seed);
    default: throw std::invalid_argument("tuner not provided by the GPU runtime (out of scope)");
  }
}

// ---------------------------------------------------------------- the loops

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// Candidates for idle evaluators.  One evaluator: ask_batch(1) per
// evaluation, the reference's ask() (tuners.cpp:52-58) — traces stay
// bit-identical.  W evaluators: one ask_batch(W) per refill, i.e. ONE
// surrogate fit per W evaluations (the k best LCB scores of that fit),
// handed out as evaluators go idle; candidates whose evaluator's device
// failed are handed out again first.  `ask_s` accumulates the host time
// spent asking (charged to each candidate of the batch in equal shares).
class Proposer {
 public:
  Proposer(Tuner& t, int batch) : t_(t), batch_(std::max(1, batch)) {}

  // next candidate (nullopt: space exhausted); `budget` caps a refill
  std::optional<std::uint64_t> next(std::uint64_t budget, double* ask_share) {
    *ask_share = 0.0;
    if (!requeue_.empty()) {
      const auto f = requeue_.front();
      requeue_.pop_front();
      return f;
    }
    if (buf_.empty()) {
      const int k = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(batch_, budget)));
      const auto t0 = Clock::now();
      const auto got = t_.ask_batch(k);
      const double dt = secs(t0, Clock::now());
      ask_s_ += dt;
      if (got.empty()) return std::nullopt;
      share_ = dt / static_cast<double>(got.size());
      buf_.assign(got.begin(), got.end());
    }
    const auto f = buf_.front();
    buf_.pop_front();
    *ask_share = share_;
    return f;
  }
  void requeue(std::uint64_t f) { requeue_.push_back(f); }
  double ask_s() const { return ask_s_; }

 private:
  Tuner& t_;
  int batch_;
  std::deque<std::uint64_t> buf_, requeue_;
  double share_ = 0.0, ask_s_ = 0.0;
};

}  // namespace

std::vector<Record> run_tuning_synthetic(const TuneOptions& opt, double* total_s) {
  if (opt.max_evals < 1) throw std::invalid_argument("run_tuning: max_evals must be >= 1");
  const Space space = build_space(opt.kernel, opt.size);
  auto tuner = make_tuner(opt.tuner, space, opt.seed);
  const int W = std::max(1, opt.workers);
  Proposer prop(*tuner, W);
  // discrete-event simulation: (finish time, issue order, worker, flat)
  using Ev = std::tuple<double, std::uint64_t, int, std::uint64_t>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> running;
  std::vector<Record> recs;
  double now = 0.0, best = std::numeric_limits<double>::infinity();
  std::uint64_t issued = 0;
  std::vector<int> idle;
  for (int w = W - 1; w >= 0; --w) idle.push_back(w);
  auto dispatch = [&] {
    while (!idle.empty() && recs.size() + running.size() < opt.max_evals &&
           !(opt.max_seconds && now >= *opt.max_seconds)) {
      double share;
      const auto got = prop.next(opt.max_evals - recs.size() - running.size(), &share);
      if (!got) break;
      const int w = idle.back();
      idle.pop_back();
      const double rt = synthetic_objective(space, config_at(space, *got));
      running.emplace(now + rt, issued++, w, *got);
    }
  };
  dispatch();
  while (!running.empty()) {
    auto [fin, ord, w, flat] = running.top();
    (void)ord;
    running.pop();
    now = fin;
    const auto cfg = config_at(space, flat);
    const double rt = synthetic_objective(space, cfg);
    tuner->tell(flat, rt);
    best = std::min(best, rt);
    recs.push_back({recs.size(), flat, cfg, rt, now, best, w, 0.0, rt});
    idle.push_back(w);
    dispatch();
  }
  if (total_s) *total_s = now;
  return recs;
}

std::vector<Record> run_tuning(const TuneOptions& opt, const Objective& objective,
                               double* total_s, std::string* error) {
  if (opt.max_evals < 1) throw std::invalid_argument("run_tuning: max_evals must be >= 1");
  const Space space = build_space(opt.kernel, opt.size);
  auto tuner = make_tuner(opt.tuner, space, opt.seed);
  const int W = std::max(1, opt.workers);
  Proposer prop(*tuner, W);

  struct Job {
    std::uint64_t flat;
    double ask_s;
  };
  struct Done {
    int worker;
    std::uint64_t flat;
    std::optional<double> rt;
    bool error;
    std::string what;
    double ask_s, eval_s;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Done> done;
  std::vector<std::optional<Job>> job(W);
  std::vector<bool> dead(W, false);
  bool stop = false;

  std::vector<std::thread> threads;
  for (int w = 0; w < W; ++w) {
    threads.emplace_back([&, w] {
      for (;;) {
        Job jb;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return stop || job[w].has_value(); });
          if (stop && !job[w]) return;
          jb = *job[w];
        }
        Done d{w, jb.flat, std::nullopt, false, {}, jb.ask_s, 0.0};
        const auto t0 = Clock::now();
        try {
          d.rt = objective(w, config_at(space, jb.flat));
        } catch (const std::exception& e) {
          d.error = true;
          d.what = e.what();
        }
        d.eval_s = secs(t0, Clock::now());
        {
          std::lock_guard<std::mutex> lk(mu);
          job[w].reset();
          done.push_back(std::move(d));
        }
        cv.notify_all();
      }
    });
  }

  const auto start = Clock::now();
  auto elapsed = [&] { return secs(start, Clock::now()); };
  std::vector<Record> recs;
  double best = std::numeric_limits<double>::infinity();
  int in_flight = 0, alive = W;
  std::string first_error;
  bool exhausted = false;
  {
    std::unique_lock<std::mutex> lk(mu);
    auto dispatch = [&] {
      for (int w = 0; w < W; ++w) {
        if (job[w] || dead[w] || exhausted) continue;
        if (recs.size() + in_flight >= opt.max_evals) return;
        if (opt.max_seconds && elapsed() >= *opt.max_seconds) return;  // checked before each eval
        double share;
        const auto got = prop.next(opt.max_evals - recs.size() - in_flight, &share);
        if (!got) {
          exhausted = true;
          return;
        }
        job[w] = Job{*got, share};
        ++in_flight;
      }
    };
    dispatch();
    cv.notify_all();
    while (in_flight > 0) {
      cv.wait(lk, [&] { return !done.empty(); });
      while (!done.empty()) {
        Done d = std::move(done.front());
        done.pop_front();
        --in_flight;
        if (d.error) {
          // MeasurementError on this evaluator's device (harness.cpp:252-256):
          // the evaluator is retired and its candidate handed to another one;
          // with none left the run stops and returns the partial trace.
          if (first_error.empty()) first_error = d.what;
          dead[d.worker] = true;
          --alive;
          prop.requeue(d.flat);
          continue;
        }
        tuner->tell(d.flat, d.rt);
        if (d.rt) best = std::min(best, *d.rt);
        recs.push_back({recs.size(), d.flat, config_at(space, d.flat), d.rt, elapsed(), best,
                        d.worker, d.ask_s, d.eval_s});
      }
      if (alive > 0) dispatch();
      cv.notify_all();
    }
    stop = true;
  }
  cv.notify_all();
  for (auto& t : threads) t.join();
  if (total_s) *total_s = elapsed();
  if (error) {
    error->clear();
    if (alive == 0) *error = first_error;  // every evaluator failed: the run is incomplete
  } else if (alive == 0) {
    throw std::runtime_error(first_error);
  }
  return recs;
}

std::vector<Record> run_tuning_virtual(const TuneOptions& opt, const VirtualObjective& objective,
                                       double* total_s, std::string* error) {
  if (opt.max_evals < 1) throw std::invalid_argument("run_tuning: max_evals must be >= 1");
  const Space space = build_space(opt.kernel, opt.size);
  auto tuner = make_tuner(opt.tuner, space, opt.seed);
  const int W = std::max(1, opt.workers);
  Proposer prop(*tuner, W);
  struct Ev {
    double fin;
    std::uint64_t ord;
    int worker;
    std::uint64_t flat;
    std::optional<double> rt;
    double ask_s, eval_s;
    bool operator>(const Ev& o) const { return fin != o.fin ? fin > o.fin : ord > o.ord; }
  };
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> running;
  std::vector<Record> recs;
  double now = 0.0, disp = 0.0, best = std::numeric_limits<double>::infinity();
  std::uint64_t issued = 0;
  std::vector<int> idle;
  for (int w = W - 1; w >= 0; --w) idle.push_back(w);
  std::string err;
  // the dispatcher is one host thread: asks are serial on the virtual clock
  auto dispatch = [&] {
    while (!idle.empty() && err.empty() && recs.size() + running.size() < opt.max_evals) {
      const double t_ask = std::max(now, disp);
      if (opt.max_seconds && t_ask >= *opt.max_seconds) break;
      const double before = prop.ask_s();
      double share;
      const auto got = prop.next(opt.max_evals - recs.size() - running.size(), &share);
      disp = t_ask + (prop.ask_s() - before);  // the real host time of this ask
      if (!got) break;
      const int w = idle.back();
      idle.pop_back();
      std::pair<std::optional<double>, double> r;
      try {
        r = objective(config_at(space, *got));  // measured now, revealed at its finish time
      } catch (const std::exception& e) {
        err = e.what();  // the one real device failed: every virtual evaluator is gone
        break;
      }
      running.push({disp + r.second, issued++, w, *got, r.first, share, r.second});
    }
  };
  dispatch();
  while (!running.empty()) {
    Ev e = running.top();
    running.pop();
    now = e.fin;
    tuner->tell(e.flat, e.rt);
    if (e.rt) best = std::min(best, *e.rt);
    recs.push_back({recs.size(), e.flat, config_at(space, e.flat), e.rt, now, best, e.worker,
                    e.ask_s, e.eval_s});
    idle.push_back(e.worker);
    dispatch();
  }
  if (total_s) *total_s = now;
  if (error) *error = err;
  return recs;
}

}  // namespace tth
