// TEST INFRASTRUCTURE ONLY — a standalone driver over the UNMODIFIED
// reference core (oracle/_ref/libtiletuner_ref.so) for the CLI tests:
//   ref_trace render <kernel> <size> <tuner> <seed> <max_evals>
//       run_tuning with the synthetic objective (harness.cpp:199-265),
//       created = 0 as the CLI's --reproducible (tiletuner.cpp:166), and
//       render_trace (persist.cpp:97-127) to stdout;
//   ref_trace parse <file>
//       read_trace (persist.cpp:129-230) + best_of: "<records> <config> <best>".
// A separate process because the reference's iostream code must not share
// a process with another libstdc++ (the Python test runner's).
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>

#include "tiletuner/harness.hpp"
#include "tiletuner/persist.hpp"
#include "tiletuner/problem.hpp"
#include "tiletuner/space.hpp"
#include "tiletuner/tuners.hpp"

using namespace tiletuner;

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "render" && argc == 7) {
      const ParamSpace space = build_space(parse_kernel(argv[2]), argv[3]);
      Budget budget;
      budget.max_evals = std::strtoull(argv[6], nullptr, 10);
      TuningTrace t = run_tuning(parse_tuner(argv[4]), space, SyntheticObjective{}, budget,
                                 MeasureProtocol{}, std::strtoull(argv[5], nullptr, 10));
      t.created_unix = 0;
      std::cout << render_trace(t);
      return 0;
    }
    if (cmd == "parse" && argc == 3) {
      const TuningTrace t = read_trace(argv[2]);
      const auto best = best_of(t);
      char b[40];
      std::snprintf(b, sizeof b, "%.17g", best.second);
      std::cout << t.records.size() << ' ' << format_config(best.first) << ' ' << b << '\n';
      return 0;
    }
    std::cerr << "usage: ref_trace render <kernel> <size> <tuner> <seed> <evals> | parse <file>\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
