/* tt_tuner.h — C ABI of the host-side tuning runtime (libtt_tuner.so).
 *
 * Replaces the reference's in-process C++ tuning stack on the path to the
 * GPU objective (/root/reference/proj/core/include/tiletuner/space.hpp,
 * tuners.hpp, harness.hpp):
 *   - the tile-factor search space, bit-exact with space.cpp:10-124
 *     (divisor candidates, mixed-radix flat index, log2 encoding);
 *   - ask/tell tuners (random, grid, bayesopt = random forest + LCB,
 *     tuners.cpp:131-139, :324-351) with a batch extension: a SET of pending
 *     configurations, ask_batch(1) consuming the RNG exactly like ask();
 *   - run_tuning (harness.cpp:199-265): synthetic objective on a virtual
 *     clock, or the measured GPU objective with one worker thread and one
 *     tt_ctx per device, dispatching a new candidate to each device as soon
 *     as it is idle.
 * Kernel ids follow tt_gpu.h; tuner ids follow tiletuner::TunerKind
 * (random 0, grid 1, genetic 2, boosted 3, bayesopt 4; 2 and 3 are not
 * provided and return TT_EINVAL).  Status codes are those of tt_gpu.h.
 */
#ifndef TT_TUNER_H
#define TT_TUNER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t eval_index;
  uint64_t flat;
  int config[6];
  int nconfig;
  int failed;          /* 1: NumericalError, runtime_s is undefined */
  double runtime_s;
  double elapsed_s;    /* since the clock started (virtual for synthetic runs) */
  double best_so_far_s;
  int worker;          /* evaluator (device slot) that measured it */
  double ask_s;        /* host time spent asking for it (its share of a batch ask) */
  double eval_s;       /* wall time of its evaluation */
} tt_record;

/* ---- search space (space.hpp:41-68) ---- */
int tt_space_divisors(int n, int* out, int cap); /* returns the count, -1 on error */
int tt_space_size(int kernel, const char* size, uint64_t* out);
int tt_space_config_at(int kernel, const char* size, uint64_t flat, int* cfg);
int tt_space_index_of(int kernel, const char* size, const int* cfg, int ncfg, uint64_t* out);
int tt_space_encode(int kernel, const char* size, const int* cfg, int ncfg, double* out);
int tt_space_synthetic(int kernel, const char* size, const int* cfg, int ncfg, double* out);

/* ---- ask/tell handle ---- */
typedef struct tt_tuner tt_tuner;
int tt_tuner_create(int tuner, int kernel, const char* size, uint64_t seed, tt_tuner** out);
int tt_tuner_ask_batch(tt_tuner* t, int k, uint64_t* flats, int* got);
int tt_tuner_tell(tt_tuner* t, uint64_t flat, int failed, double runtime_s);
int tt_tuner_destroy(tt_tuner* t);

/* ---- run_tuning ---- */
/* Synthetic objective, `workers` simulated evaluators (discrete events on a
 * virtual clock).  workers = 1 reproduces the reference trace exactly.
 * max_seconds <= 0 means no wall-clock bound. */
int tt_tune_synthetic(int tuner, int kernel, const char* size, uint64_t seed, int max_evals,
                      double max_seconds, int workers, tt_record* out, int cap, int* n_out,
                      double* total_s);

/* Measured objective on the GPUs: one worker per entry of `devices`, inputs
 * generated on every device from `input_seed` before the clock starts, the
 * reference's spot check (mini size, config_at(space, size/2), residual <=
 * 1e-10) first when `spot_check`, then tt_measure with the protocol.  With
 * several devices the surrogate is fitted once per batch of n_devices
 * candidates, handed out as devices go idle.  A device failure
 * (MeasurementError) retires that worker and its candidate is re-evaluated
 * on another device; when every worker failed the call returns TT_EDEVICE
 * with the partial trace in out / *n_out (harness.cpp:252-256 flushes the
 * partial trace before rethrowing).  Test hook: TT_FAULT_INJECT="w:n" makes
 * worker w fail at its n-th evaluation (0-based). */
int tt_tune_measured(int tuner, int kernel, const char* size, uint64_t seed,
                     uint64_t input_seed, int max_evals, double max_seconds,
                     const int* devices, int n_devices, int warmups, int reps, int aggregate,
                     int spot_check, tt_record* out, int cap, int* n_out, double* total_s,
                     char* err, int errcap);

/* Virtual-clock measured run (the T1 / T8 time-to-best harness): n_virtual
 * evaluators emulated on ONE real device.  Every candidate is measured for
 * real (tt_measure) and occupies its virtual evaluator for the wall time the
 * evaluation took; the real host ask time is charged serially; results reach
 * the tuner at their virtual finish time.  elapsed_s is virtual time. */
int tt_tune_virtual(int tuner, int kernel, const char* size, uint64_t seed, uint64_t input_seed,
                    int max_evals, double max_seconds, int device, int n_virtual, int warmups,
                    int reps, int aggregate, int spot_check, tt_record* out, int cap, int* n_out,
                    double* total_s, char* err, int errcap);

#ifdef __cplusplus
}
#endif
#endif /* TT_TUNER_H */
