// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// Thin extern "C" shim compiled together with the reference hexplan sources
// (/root/reference/proj/src/*.cpp) into oracle/_ref/libhexplan_ref.so by
// oracle/Makefile.  The reference C ABI (proj/include/hexplan.h:63-127) can
// only *produce* plans; it has no entry point that checks or prices a
// caller-supplied plan.  This shim adds exactly that, by calling the
// reference's own C++ functions:
//   * PipelinePlan::num_micro_batches        proj/src/types.hpp:70-72
//   * build_dp_groups                        proj/src/cost_model.cpp:155-164
//   * validate_plan                          proj/src/cost_model.cpp:166-208
//   * iteration_time / model_flops_utilization proj/src/cost_model.cpp:210-265
//   * serialize_plan                         proj/src/report.cpp:62-64
// so the executor's integer bookkeeping can be compared bit-exactly with the
// reference on the same plan documents.  The plan JSON -> ExecutionPlan
// conversion below is ours (the reference has no plan parser).
#include <cstdlib>
#include <cstring>
#include <string>

#include "cost_model.hpp"
#include "errors.hpp"
#include "json.hpp"
#include "json_io.hpp"
#include "report.hpp"
#include "types.hpp"

using ojson = nlohmann::ordered_json;

namespace {

void put_err(char* err, size_t n, const std::string& m) {
  if (!err || n == 0) return;
  size_t k = m.size() < n - 1 ? m.size() : n - 1;
  std::memcpy(err, m.data(), k);
  err[k] = '\0';
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

int device_of(const ojson& v, const hexplan::ClusterSpec& c) {
  if (v.is_string()) {
    int i = c.device_index(v.get<std::string>());
    if (i < 0) throw hexplan::ParseError("plan: unknown device id " + v.get<std::string>());
    return i;
  }
  return v.get<int>();
}

hexplan::ExecutionPlan plan_from_json(const std::string& text,
                                      const hexplan::ClusterSpec& c,
                                      bool* had_dp_groups) {
  ojson j = ojson::parse(text, nullptr, false);
  if (j.is_discarded()) throw hexplan::ParseError("plan: not valid JSON");
  if (j.contains("plan") && j["plan"].is_object()) j = j["plan"];
  hexplan::ExecutionPlan p;
  p.global_batch = j.at("global_batch").get<std::int64_t>();
  for (const auto& jp : j.at("pipelines")) {
    hexplan::PipelinePlan pp;
    pp.batch = jp.at("batch").get<std::int64_t>();
    pp.micro_batch = jp.at("micro_batch").get<std::int64_t>();
    for (const auto& js : jp.at("stages")) {
      hexplan::StagePlan st;
      for (const auto& d : js.at("devices")) st.devices.push_back(device_of(d, c));
      st.tp = js.at("tp").get<int>();
      st.layer_start = js.at("layer_start").get<int>();
      st.layer_count = js.at("layer_count").get<int>();
      pp.stages.push_back(std::move(st));
    }
    p.pipelines.push_back(std::move(pp));
  }
  *had_dp_groups = j.contains("dp_groups");
  if (*had_dp_groups) {
    for (const auto& jg : j["dp_groups"]) {
      hexplan::DpGroup g;
      g.layer = jg.at("layer").get<int>();
      for (const auto& d : jg.at("members")) g.members.push_back(device_of(d, c));
      p.dp_groups.push_back(std::move(g));
    }
  }
  return p;
}

ojson ids(const std::vector<int>& v, const hexplan::ClusterSpec& c) {
  ojson a = ojson::array();
  for (int i : v)
    a.push_back(i >= 0 && i < int(c.devices.size()) ? ojson(c.devices[i].id) : ojson(i));
  return a;
}

}  // namespace

extern "C" {

// Returns 0 and a malloc'd JSON report in *out on success; non-zero on a
// parse failure of the inputs (err filled).  Plan-invariant violations are
// reported inside the JSON ("validate"), like the reference reports them
// through InvalidArgument messages.
int hexref_check_plan(const char* cluster_json, const char* model_json,
                      const char* plan_json, char** out, char* err,
                      size_t err_len) {
  try {
    hexplan::ClusterSpec c = hexplan::parse_cluster(cluster_json);
    hexplan::ModelSpec m = hexplan::parse_model(model_json);
    bool had = false;
    hexplan::ExecutionPlan plan = plan_from_json(plan_json, c, &had);
    ojson r;
    r["num_micro_batches"] = ojson::array();
    for (const auto& p : plan.pipelines) r["num_micro_batches"].push_back(p.num_micro_batches());
    hexplan::ExecutionPlan rebuilt = plan;
    // the reference build_dp_groups reads stage.devices[0] unchecked; skip it for
    // stage-less-device plans (validate_plan rejects them anyway)
    bool any_empty = false;
    for (const auto& p : plan.pipelines)
      for (const auto& st : p.stages)
        any_empty |= st.devices.empty() || st.layer_start < 0 ||
                     st.layer_start + st.layer_count > m.num_layers;
    if (!any_empty) hexplan::build_dp_groups(rebuilt, m);
    r["dp_groups"] = ojson::array();
    for (const auto& g : rebuilt.dp_groups)
      r["dp_groups"].push_back({{"layer", g.layer}, {"members", ids(g.members, c)}});
    if (!had) plan.dp_groups = rebuilt.dp_groups;
    try {
      hexplan::validate_plan(plan, m, c);
      r["validate"] = "ok";
    } catch (const std::exception& e) {
      r["validate"] = e.what();
    }
    if (r["validate"] == "ok") try {
      hexplan::CostReport rep = hexplan::iteration_time(plan, m, c, 1.0);
      r["cost"] = ojson::parse(hexplan::serialize_report(rep, c));
    } catch (const std::exception& e) {
      r["cost_error"] = e.what();
    }
    if (r["validate"] == "ok") r["plan_serialized"] = hexplan::serialize_plan(plan, c);
    *out = dup(r.dump());
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// MFU in the reference convention (cost_model.cpp:260-265) for a measured
// iteration time; returns 0 on bad input.
double hexref_mfu(const char* cluster_json, const char* model_json,
                  double seconds, long long global_batch) {
  try {
    hexplan::ClusterSpec c = hexplan::parse_cluster(cluster_json);
    hexplan::ModelSpec m = hexplan::parse_model(model_json);
    return hexplan::model_flops_utilization(seconds, global_batch, m, c);
  } catch (...) {
    return 0.0;
  }
}

void hexref_free(char* s) { std::free(s); }

}  // extern "C"
