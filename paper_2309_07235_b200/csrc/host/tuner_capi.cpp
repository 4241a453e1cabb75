// C ABI of the host tuning runtime (include/tt_tuner.h).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "../../../include/tt_gpu.h"
#include "../../../include/tt_tuner.h"
#include "tuner.hpp"

using namespace tth;

struct tt_tuner {
  std::unique_ptr<Tuner> impl;
};

namespace {

Kernel kernel_of(int k) {
  if (k < 0 || k > 2) throw std::invalid_argument("unknown kernel id");
  return static_cast<Kernel>(k);
}

template <class F>
int guarded(F&& f, std::string* err = nullptr) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    if (err) *err = e.what();
    return TT_EINVAL;
  } catch (const std::out_of_range& e) {
    if (err) *err = e.what();
    return TT_EINVAL;
  } catch (const std::exception& e) {
    if (err) *err = e.what();
    return TT_EDEVICE;
  }
}

void fill(const std::vector<Record>& recs, tt_record* out, int cap, int* n_out) {
  const int n = static_cast<int>(recs.size());
  if (n_out) *n_out = n;
  for (int i = 0; i < n && i < cap; ++i) {
    tt_record& r = out[i];
    std::memset(&r, 0, sizeof r);
    r.eval_index = recs[i].eval_index;
    r.flat = recs[i].flat;
    r.nconfig = static_cast<int>(recs[i].config.size());
    for (int j = 0; j < r.nconfig && j < 6; ++j) r.config[j] = recs[i].config[j];
    r.failed = recs[i].runtime_s ? 0 : 1;
    r.runtime_s = recs[i].runtime_s ? *recs[i].runtime_s : 0.0;
    r.elapsed_s = recs[i].elapsed_s;
    r.best_so_far_s = recs[i].best_so_far_s;
    r.worker = recs[i].worker;
    r.ask_s = recs[i].ask_s;
    r.eval_s = recs[i].eval_s;
  }
}

std::vector<int> cfgv(const int* cfg, int n) { return std::vector<int>(cfg, cfg + n); }

// Host oracle-free reference for the 3mm spot check: naive i,j,k products
// (kernels.cpp:73-86 shape) of the mini inputs downloaded from the device.
std::vector<double> naive_mm(const std::vector<double>& x, const std::vector<double>& y, int r,
                             int k, int c) {
  std::vector<double> o(static_cast<size_t>(r) * c, 0.0);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) {
      double acc = 0.0;
      for (int t = 0; t < k; ++t) acc += x[static_cast<size_t>(i) * k + t] * y[static_cast<size_t>(t) * c + j];
      o[static_cast<size_t>(i) * c + j] = acc;
    }
  return o;
}

struct Ctx {
  tt_ctx* h = nullptr;
  ~Ctx() {
    if (h) tt_ctx_destroy(h);
  }
};

void check(tt_ctx* c, int rc, const char* what) {
  if (rc == TT_OK) return;
  std::string msg = std::string(what) + ": " + tt_last_error(c);
  if (rc == TT_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// harness.cpp:147-156 on the GPU path
void spot_check(tt_ctx* c, Kernel k) {
  const ProblemSize* mini = find_size(k, "mini");
  const Space sp = build_space(k, "mini");
  const std::vector<int> probe = config_at(sp, sp.size() / 2);
  check(c, tt_setup_seeded(c, static_cast<int>(k), mini->n, mini->l, mini->m, mini->o, mini->p, 1),
        "spot check setup");
  std::vector<double> out(static_cast<size_t>(mini->n) * (k == Kernel::mm3 ? mini->p : mini->n));
  int fail = -1;
  check(c, tt_run(c, probe.data(), static_cast<int>(probe.size()), out.data(), &fail),
        "spot check run");
  double res = 0.0;
  if (k == Kernel::mm3) {
    std::vector<double> A(static_cast<size_t>(mini->n) * mini->l), B(static_cast<size_t>(mini->l) * mini->m),
        C(static_cast<size_t>(mini->m) * mini->o), D(static_cast<size_t>(mini->o) * mini->p);
    check(c, tt_get_input(c, A.data(), B.data(), C.data(), D.data()), "spot check inputs");
    const auto E = naive_mm(A, B, mini->n, mini->l, mini->m);
    const auto F = naive_mm(C, D, mini->m, mini->o, mini->p);
    const auto G = naive_mm(E, F, mini->n, mini->m, mini->p);
    check(c, tt_residual(c, G.data(), &res), "spot check residual");
  } else {
    check(c, tt_residual(c, nullptr, &res), "spot check residual");
  }
  if (!(res <= 1e-10))
    throw std::runtime_error("spot check failed: tiled kernel residual " + std::to_string(res));
}

}  // namespace

extern "C" {

int tt_space_divisors(int n, int* out, int cap) {
  if (n < 1) return -1;
  const auto d = divisor_candidates(n);
  for (int i = 0; i < static_cast<int>(d.size()) && i < cap; ++i) out[i] = d[i];
  return static_cast<int>(d.size());
}

int tt_space_size(int kernel, const char* size, uint64_t* out) {
  return guarded([&] {
    *out = build_space(kernel_of(kernel), size).size();
    return TT_OK;
  });
}

int tt_space_config_at(int kernel, const char* size, uint64_t flat, int* cfg) {
  return guarded([&] {
    const auto c = config_at(build_space(kernel_of(kernel), size), flat);
    for (size_t i = 0; i < c.size(); ++i) cfg[i] = c[i];
    return TT_OK;
  });
}

int tt_space_index_of(int kernel, const char* size, const int* cfg, int ncfg, uint64_t* out) {
  return guarded([&] {
    return index_of(build_space(kernel_of(kernel), size), cfgv(cfg, ncfg), out) ? TT_OK
                                                                                : TT_EINVAL;
  });
}

int tt_space_encode(int kernel, const char* size, const int* cfg, int ncfg, double* out) {
  return guarded([&] {
    const auto e = encode(build_space(kernel_of(kernel), size), cfgv(cfg, ncfg));
    for (size_t i = 0; i < e.size(); ++i) out[i] = e[i];
    return TT_OK;
  });
}

int tt_space_synthetic(int kernel, const char* size, const int* cfg, int ncfg, double* out) {
  return guarded([&] {
    const Space sp = build_space(kernel_of(kernel), size);
    std::uint64_t tmp;
    if (!index_of(sp, cfgv(cfg, ncfg), &tmp)) return TT_EINVAL;
    *out = synthetic_objective(sp, cfgv(cfg, ncfg));
    return TT_OK;
  });
}

int tt_tuner_create(int tuner, int kernel, const char* size, uint64_t seed, tt_tuner** out) {
  return guarded([&] {
    auto t = std::make_unique<tt_tuner>();
    t->impl = make_tuner(static_cast<TunerKind>(tuner), build_space(kernel_of(kernel), size), seed);
    *out = t.release();
    return TT_OK;
  });
}

int tt_tuner_ask_batch(tt_tuner* t, int k, uint64_t* flats, int* got) {
  return guarded([&] {
    const auto v = t->impl->ask_batch(k);
    for (size_t i = 0; i < v.size(); ++i) flats[i] = v[i];
    *got = static_cast<int>(v.size());
    return TT_OK;
  });
}

int tt_tuner_tell(tt_tuner* t, uint64_t flat, int failed, double runtime_s) {
  return guarded([&] {
    t->impl->tell(flat, failed ? std::nullopt : std::optional<double>(runtime_s));
    return TT_OK;
  });
}

int tt_tuner_destroy(tt_tuner* t) {
  delete t;
  return TT_OK;
}

int tt_tune_synthetic(int tuner, int kernel, const char* size, uint64_t seed, int max_evals,
                      double max_seconds, int workers, tt_record* out, int cap, int* n_out,
                      double* total_s) {
  return guarded([&] {
    TuneOptions o;
    o.tuner = static_cast<TunerKind>(tuner);
    o.kernel = kernel_of(kernel);
    o.size = size;
    o.seed = seed;
    o.max_evals = static_cast<std::uint64_t>(max_evals);
    if (max_seconds > 0) o.max_seconds = max_seconds;
    o.workers = workers;
    fill(run_tuning_synthetic(o, total_s), out, cap, n_out);
    return TT_OK;
  });
}

namespace {

// TT_FAULT_INJECT="w:n": worker w fails (MeasurementError) at its n-th evaluation.
struct FaultPlan {
  int worker = -1, at = -1;
};
FaultPlan fault_plan() {
  FaultPlan f;
  if (const char* v = std::getenv("TT_FAULT_INJECT")) std::sscanf(v, "%d:%d", &f.worker, &f.at);
  return f;
}

void copy_err(const std::string& msg, char* err, int errcap) {
  if (err && errcap > 0) {
    std::strncpy(err, msg.c_str(), static_cast<size_t>(errcap) - 1);
    err[errcap - 1] = '\0';
  }
}

TuneOptions options(int tuner, Kernel k, const char* size, uint64_t seed, int max_evals,
                    double max_seconds, int workers) {
  TuneOptions o;
  o.tuner = static_cast<TunerKind>(tuner);
  o.kernel = k;
  o.size = size;
  o.seed = seed;
  o.max_evals = static_cast<std::uint64_t>(max_evals);
  if (max_seconds > 0) o.max_seconds = max_seconds;
  o.workers = workers;
  return o;
}

}  // namespace

int tt_tune_measured(int tuner, int kernel, const char* size, uint64_t seed, uint64_t input_seed,
                     int max_evals, double max_seconds, const int* devices, int n_devices,
                     int warmups, int reps, int aggregate, int spot, tt_record* out, int cap,
                     int* n_out, double* total_s, char* err, int errcap) {
  std::string msg;
  if (n_out) *n_out = 0;
  const int rc = guarded(
      [&] {
        if (n_devices < 1) throw std::invalid_argument("need at least one device");
        if (warmups < 0 || reps < 1)
          throw std::invalid_argument("measure: warmups must be >= 0 and repetitions >= 1");
        const Kernel k = kernel_of(kernel);
        const ProblemSize* ps = find_size(k, size);
        if (!ps) throw std::out_of_range(std::string("unregistered problem size: ") + size);
        std::vector<Ctx> ctxs(n_devices);
        // contexts + inputs on every device before the clock starts (harness.cpp:220-227)
        std::vector<std::string> errs(n_devices);
        std::vector<std::thread> th;
        for (int w = 0; w < n_devices; ++w) {
          th.emplace_back([&, w] {
            try {
              if (tt_ctx_create(devices[w], &ctxs[w].h) != TT_OK)
                throw std::runtime_error("tt_ctx_create failed on device " +
                                         std::to_string(devices[w]));
              if (spot && w == 0) spot_check(ctxs[w].h, k);
              check(ctxs[w].h,
                    tt_setup_seeded(ctxs[w].h, kernel, ps->n, ps->l, ps->m, ps->o, ps->p,
                                    input_seed),
                    "setup");
            } catch (const std::exception& e) {
              errs[w] = e.what();
            }
          });
        }
        for (auto& t : th) t.join();
        for (auto& e : errs)
          if (!e.empty()) throw std::runtime_error(e);
        const FaultPlan fp = fault_plan();
        std::vector<int> evals(n_devices, 0);  // per worker (each touched by its own thread)
        Objective obj = [&](int w, const std::vector<int>& cfg) -> std::optional<double> {
          if (w == fp.worker && evals[w]++ == fp.at)
            throw std::runtime_error("injected device fault on worker " + std::to_string(w));
          double secs = 0.0;
          const int r = tt_measure(ctxs[w].h, cfg.data(), static_cast<int>(cfg.size()), warmups,
                                   reps, aggregate, &secs);
          if (r == TT_ENUMERIC) return std::nullopt;  // penalised failure (harness.cpp:250-251)
          check(ctxs[w].h, r, "measure");              // MeasurementError: worker retired
          return secs;
        };
        std::string run_err;
        const auto recs = run_tuning(options(tuner, k, size, seed, max_evals, max_seconds, n_devices),
                                     obj, total_s, &run_err);
        fill(recs, out, cap, n_out);  // the (partial) trace is returned either way
        if (!run_err.empty()) throw std::runtime_error("measurement error: " + run_err);
        return TT_OK;
      },
      &msg);
  if (rc != TT_OK) copy_err(msg, err, errcap);
  return rc;
}

int tt_tune_virtual(int tuner, int kernel, const char* size, uint64_t seed, uint64_t input_seed,
                    int max_evals, double max_seconds, int device, int n_virtual, int warmups,
                    int reps, int aggregate, int spot, tt_record* out, int cap, int* n_out,
                    double* total_s, char* err, int errcap) {
  std::string msg;
  if (n_out) *n_out = 0;
  const int rc = guarded(
      [&] {
        if (n_virtual < 1) throw std::invalid_argument("need at least one evaluator");
        if (warmups < 0 || reps < 1)
          throw std::invalid_argument("measure: warmups must be >= 0 and repetitions >= 1");
        const Kernel k = kernel_of(kernel);
        const ProblemSize* ps = find_size(k, size);
        if (!ps) throw std::out_of_range(std::string("unregistered problem size: ") + size);
        Ctx c;
        if (tt_ctx_create(device, &c.h) != TT_OK)
          throw std::runtime_error("tt_ctx_create failed on device " + std::to_string(device));
        if (spot) spot_check(c.h, k);
        check(c.h, tt_setup_seeded(c.h, kernel, ps->n, ps->l, ps->m, ps->o, ps->p, input_seed),
              "setup");
        VirtualObjective obj = [&](const std::vector<int>& cfg) {
          const auto t0 = std::chrono::steady_clock::now();
          double secs = 0.0;
          const int r = tt_measure(c.h, cfg.data(), static_cast<int>(cfg.size()), warmups, reps,
                                   aggregate, &secs);
          const double wall =
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          if (r == TT_ENUMERIC) return std::make_pair(std::optional<double>(), wall);
          check(c.h, r, "measure");
          return std::make_pair(std::optional<double>(secs), wall);
        };
        std::string run_err;
        const auto recs = run_tuning_virtual(
            options(tuner, k, size, seed, max_evals, max_seconds, n_virtual), obj, total_s, &run_err);
        fill(recs, out, cap, n_out);
        if (!run_err.empty()) throw std::runtime_error("measurement error: " + run_err);
        return TT_OK;
      },
      &msg);
  if (rc != TT_OK) copy_err(msg, err, errcap);
  return rc;
}

}  // extern "C"
