// run_b200.cpp — the reference's run() call site moved onto the B200 engine
// through the header-only C++ face (include/mgfwa_b200.hpp).
//
//   g++ -std=c++17 -I include examples/run_b200.cpp \
//       -L paper_2501_03944_b200 -lmgfwa_b200 -Wl,-rpath,$PWD/paper_2501_03944_b200
//   ./a.out run        # C1: sphere D=30, B=1, mu=5, lambda=30, 1e5 evaluations
//   ./a.out validate   # host-side validation only (no GPU needed)
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "mgfwa_b200.hpp"

int main(int argc, char** argv) {
  using namespace mgfwa::b200;
  const char* mode = argc > 1 ? argv[1] : "run";
  if (std::strcmp(mode, "validate") == 0) {
    MgfwaConfig bad;
    bad.amp_amplify = 1.0;
    bad.max_evaluations = 1000;
    try {
      Engine e(bad, SearchSpace::box(4, -1.0, 1.0), Objective::sphere(), 0);
      std::printf("FAIL: no exception\n");
      return 1;
    } catch (const std::invalid_argument& ex) {
      std::printf("invalid_argument: %s\n", ex.what());
    }
    MgfwaConfig small;
    small.max_evaluations = 39;  // < B * mu = 40
    try {
      Engine e(small, SearchSpace::box(4, -1.0, 1.0), Objective::sphere(), 0);
      std::printf("FAIL: no exception\n");
      return 1;
    } catch (const std::invalid_argument& ex) {
      std::printf("invalid_argument: %s\n", ex.what());
    }
    return 0;
  }
  MgfwaConfig cfg;
  cfg.batches = 1;
  cfg.max_evaluations = 100000;
  const RunRecord r = run(cfg, SearchSpace::box(30, -10.0, 10.0), Objective::sphere(), 0);
  std::printf("evaluations %llu iterations %llu losers %llu best %.6g waves %zu\n",
              (unsigned long long)r.evaluations_used, (unsigned long long)r.iterations,
              (unsigned long long)r.losers_reinitialized, r.best_fitness[0], r.trace[0].size());
  return r.best_fitness[0] < r.trace[0].front().best_fitness ? 0 : 1;
}
