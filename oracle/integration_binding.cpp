// ORACLE TEST INFRASTRUCTURE — the INTEGRATION.md binding, compiled.
//
// What a hexplan-side maintainer adds next to proj/tools/hexplan_cli.cpp:
// the reference planner's C ABI (proj/include/hexplan.h:33-144) produces a
// plan, and hexexec's C ABI (include/hexexec.h) consumes the same documents.
// Both shared libraries are linked: oracle/_ref/libhexplan_ref.so (built from
// the reference sources by oracle/Makefile) and
// paper_2409_01143_b200/libhexexec.so.  Host only: every executor context is
// created with "validate_only" (plan ingestion, rank layout, per-rank memory
// sizing against memory_gib), so it runs without a GPU.
//
// Mirrors /root/reference/proj/tests/test_capi.cpp:55-271 (round trip through
// the C boundary, error codes, NUL-terminated truncated err buffers,
// infeasible-is-a-value, strict config keys) on the executor side.
//
//   oracle/_ref/integration_binding            -> prints one JSON line, exit 0
// Driven by tests/test_integration_binding.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "hexexec.h"
#include "hexplan.h"

namespace {

int failures = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::fprintf(stderr, "CHECK failed at line %d: %s\n", __LINE__, #cond); \
      ++failures;                                                         \
    }                                                                     \
  } while (0)

// reference test fixture (test_capi.cpp:11-29)
const char* kCluster = R"({
  "machines": {
    "A": {"intra_bandwidth_gbps": 200, "intra_latency_us": 10},
    "B": {"intra_bandwidth_gbps": 32, "intra_latency_us": 500}
  },
  "devices": [
    {"id": "a0", "machine": "A", "memory_gib": 80, "peak_tflops": 312},
    {"id": "a1", "machine": "A", "memory_gib": 80, "peak_tflops": 312},
    {"id": "b0", "machine": "B", "memory_gib": 24, "peak_tflops": 165},
    {"id": "b1", "machine": "B", "memory_gib": 24, "peak_tflops": 165}
  ],
  "inter": {"bandwidth_gbps": 12, "latency_us": 1000}
})";
const char* kModel = R"({
  "num_layers": 8, "hidden_dim": 2048, "seq_len": 2048, "bytes_per_element": 2
})";
const char* kConfig = R"({"global_batch": 16, "iterations": 8, "seed": 1, "threads": 1})";

std::string take_plan(char* s) {
  std::string out = s ? s : "";
  if (s) hexplan_string_free(s);
  return out;
}
std::string take_exec(char* s) {
  std::string out = s ? s : "";
  if (s) hexexec_string_free(s);
  return out;
}

}  // namespace

int main() {
  char err[256] = {0};
  // 1. the reference planner emits a plan through its C ABI
  hexplan_cluster* c = nullptr;
  hexplan_model* m = nullptr;
  if (hexplan_cluster_parse(kCluster, &c, err, sizeof err) != HEXPLAN_OK ||
      hexplan_model_parse(kModel, &m, err, sizeof err) != HEXPLAN_OK) {
    std::fprintf(stderr, "hexplan parse: %s\n", err);
    return 2;
  }
  hexplan_result* res = nullptr;
  CHECK(hexplan_schedule(c, m, kConfig, &res, err, sizeof err) == HEXPLAN_OK);
  CHECK(res && hexplan_result_found(res) == 1);
  const double ref_cost = res ? hexplan_result_cost(res) : 0.0;
  const std::string plan = take_plan(res ? hexplan_result_plan_json(res) : nullptr);
  const std::string cluster = take_plan(hexplan_cluster_serialize(c));
  const std::string model = take_plan(hexplan_model_serialize(m));
  CHECK(!plan.empty());

  // 2. hexexec ingests the same documents (bare plan and the CLI wrapper,
  //    hexplan_cli.cpp:217-218) and re-serializes the plan byte-identically
  hexexec_plan* p = nullptr;
  CHECK(hexexec_plan_parse(cluster.c_str(), model.c_str(), plan.c_str(), &p, err, sizeof err) ==
        HEXEXEC_OK);
  CHECK(p != nullptr);
  const std::string again = p ? take_exec(hexexec_plan_serialize(p)) : "";
  CHECK(again == plan);
  const std::string wrapped = "{\"manifest\": {\"version\": \"test\"}, \"plan\": " + plan + "}";
  hexexec_plan* pw = nullptr;
  CHECK(hexexec_plan_parse(cluster.c_str(), model.c_str(), wrapped.c_str(), &pw, err,
                           sizeof err) == HEXEXEC_OK);
  CHECK(pw && take_exec(hexexec_plan_serialize(pw)) == plan);
  if (pw) hexexec_plan_free(pw);

  // 3. the executor's restated cost model prices the plan like the reference
  //    planner did (iteration_time, cost_model.cpp:210-258; the scheduler's
  //    default state_multiplier is 1.0)
  char* report = nullptr;
  double ex_cost = -1;
  if (p && hexexec_plan_cost(p, 1.0, 0, &report, err, sizeof err) == HEXEXEC_OK && report) {
    const char* t = std::strstr(report, "\"total\":");
    if (t) ex_cost = std::strtod(t + 8, nullptr);
    hexexec_string_free(report);
  }
  CHECK(ex_cost > 0 && std::abs(ex_cost - ref_cost) <= 1e-12 * ref_cost);

  // 4. one executor context per world rank, host-only sizing (validate_only)
  const int world = p ? hexexec_plan_world_size(p) : 0;
  CHECK(world == 4);
  int created = 0;
  for (int r = 0; r < world; ++r) {
    hexexec_ctx* ctx = nullptr;
    if (hexexec_ctx_create(cluster.c_str(), model.c_str(), plan.c_str(),
                           "{\"validate_only\": true, \"seed\": 0}", r, world, r, nullptr, 0,
                           &ctx, err, sizeof err) == HEXEXEC_OK &&
        ctx) {
      const std::string st = take_exec(hexexec_stats_json(ctx));
      CHECK(st.find("\"arena_bytes\"") != std::string::npos);
      ++created;
      hexexec_ctx_free(ctx);
    } else {
      std::fprintf(stderr, "ctx_create rank %d: %s\n", r, err);
    }
  }
  CHECK(created == world);

  // 5. error conventions at the executor boundary (test_capi.cpp:71-94, :156-165)
  hexexec_ctx* bad = nullptr;
  err[0] = 0;
  CHECK(hexexec_ctx_create(cluster.c_str(), model.c_str(), plan.c_str(),
                           "{\"mystery_knob\": 1}", 0, world, 0, nullptr, 0, &bad, err,
                           sizeof err) == HEXEXEC_ERR_PARSE);
  CHECK(bad == nullptr && std::string(err).find("mystery_knob") != std::string::npos);
  CHECK(hexexec_plan_parse(nullptr, model.c_str(), plan.c_str(), &pw, err, sizeof err) ==
        HEXEXEC_ERR_INVALID);
  CHECK(hexexec_plan_parse(cluster.c_str(), model.c_str(), "not json", &pw, err, sizeof err) ==
        HEXEXEC_ERR_PARSE);
  char tiny[8];
  std::memset(tiny, 'z', sizeof tiny);
  CHECK(hexexec_plan_parse(cluster.c_str(), model.c_str(), "{", &pw, tiny, sizeof tiny) ==
        HEXEXEC_ERR_PARSE);
  CHECK(tiny[7] == '\0');
  CHECK(hexexec_ctx_create(cluster.c_str(), model.c_str(), plan.c_str(), "{}", 7, world, 0,
                           nullptr, 0, &bad, err, sizeof err) == HEXEXEC_ERR_INVALID);

  // 6. a memory tier the plan does not fit is INFEASIBLE (mem_check,
  //    cost_model.cpp:130-153, applied to the executor's arena)
  std::string starved = cluster;
  const std::string key = "\"memory_gib\": 24.0";  // hexplan_cluster_serialize's form
  for (size_t at = starved.find(key); at != std::string::npos; at = starved.find(key, at + 1))
    starved.replace(at, key.size(), "\"memory_gib\": 0.25");
  int infeasible = 0;
  for (int r = 0; r < world; ++r) {
    hexexec_ctx* ctx = nullptr;
    const int st = hexexec_ctx_create(starved.c_str(), model.c_str(), plan.c_str(),
                                      "{\"validate_only\": true}", r, world, r, nullptr, 0, &ctx,
                                      err, sizeof err);
    if (st == HEXEXEC_ERR_INFEASIBLE) ++infeasible;
    if (ctx) hexexec_ctx_free(ctx);
  }
  CHECK(infeasible >= 1);

  if (p) hexexec_plan_free(p);
  if (res) hexplan_result_free(res);
  hexplan_model_free(m);
  hexplan_cluster_free(c);
  std::printf("{\"binding\": \"%s\", \"world\": %d, \"ranks_created\": %d, "
              "\"infeasible_ranks\": %d, \"reference_cost_s\": %.12g, \"executor_cost_s\": %.12g, "
              "\"hexplan\": \"%s\", \"hexexec\": \"%s\"}\n",
              failures ? "FAIL" : "ok", world, created, infeasible, ref_cost, ex_cost,
              hexplan_version(), hexexec_version());
  return failures ? 1 : 0;
}
