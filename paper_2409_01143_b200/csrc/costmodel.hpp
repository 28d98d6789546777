// The reference's analytic step-time model (proj/src/cost_model.cpp:10-265),
// restated over hexexec's plan types so the executor can price the plan it
// runs, report predicted vs measured step time, and feed measured device
// speeds back (closed-loop calibration).
//
// iteration_time() follows the reference formula exactly (parity with the
// compiled reference at rel 1e-12: tests/test_costmodel.py), including its
// refusal of mixed-speed TP stages.  iteration_time_ext() is the labelled
// extension SURVEY §8(b) asks for: a TP stage's compute is
// max_r(w_r / sum(w) * FLOPs / c_r) over its ranks (uneven tp_widths, mixed
// device speeds); everything else is the reference formula.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "plan.hpp"

namespace hexexec {

struct MemoryReport {
  std::vector<double> per_device;
  bool fits = true;
  double worst_overage = 0;
  int worst_device = -1;
};

struct CostReport {
  std::vector<double> per_pipeline;
  double dp_comm = 0, compute = 0, tp_comm = 0, pp_comm = 0, bubble = 0;
  double total = 0, mfu = 0;
  bool feasible = false;
  MemoryReport memory;
};

// cost_model.cpp:16-21: 96 * batch * S * H^2 * (1 + S / 6H)
double layer_flops(const Model& m, double batch);
// cost_model.cpp:260-265
double model_flops_utilization(double seconds, int64_t global_batch, const Model& m,
                               const Cluster& c);
// cost_model.cpp:210-258; extension=true prices uneven / mixed-speed TP stages
CostReport iteration_time(const Plan& plan, const Model& m, const Cluster& c,
                          double state_multiplier, bool extension = false);
// report.cpp:66-93 field order
std::string serialize_report(const CostReport& r, const Cluster& c);

}  // namespace hexexec
