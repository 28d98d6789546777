// Plan ingestion + integer bookkeeping (see plan.hpp).
//
// Reference semantics restated (not copied) from:
//   cluster / model documents  proj/src/json_io.cpp:80-191 (units, required keys)
//   plan wire format           proj/src/report.cpp:25-53
//   build_dp_groups            proj/src/cost_model.cpp:155-164
//   validate_plan              proj/src/cost_model.cpp:166-208 (same messages)
//   num_micro_batches          proj/src/types.hpp:70-72
#include "plan.hpp"

#include <algorithm>
#include <map>
#include <set>

#include "nlohmann/json.hpp"

namespace hexexec {

using ojson = nlohmann::ordered_json;

namespace {

ojson parse_text(const std::string& text, const char* what) {
  ojson j = ojson::parse(text, nullptr, false);
  if (j.is_discarded()) throw ParseError(std::string(what) + ": not valid JSON");
  return j;
}

double positive(const ojson& j, const char* key, const char* ctx) {
  if (!j.contains(key) || !j[key].is_number())
    throw ParseError(std::string(ctx) + ": missing numeric field '" + key + "'");
  double v = j[key].get<double>();
  if (!(v > 0)) throw ParseError(std::string(ctx) + ": '" + key + "' must be positive");
  return v;
}

double nonneg(const ojson& j, const char* key, const char* ctx) {
  if (!j.contains(key) || !j[key].is_number())
    throw ParseError(std::string(ctx) + ": missing numeric field '" + key + "'");
  double v = j[key].get<double>();
  if (v < 0) throw ParseError(std::string(ctx) + ": '" + key + "' must be >= 0");
  return v;
}

int64_t posint(const ojson& j, const char* key, const char* ctx) {
  if (!j.contains(key) || !j[key].is_number_integer())
    throw ParseError(std::string(ctx) + ": missing integer field '" + key + "'");
  int64_t v = j[key].get<int64_t>();
  if (v <= 0) throw ParseError(std::string(ctx) + ": '" + key + "' must be positive");
  return v;
}

int64_t opt_posint(const ojson& j, const char* key, int64_t dflt, const char* ctx) {
  if (!j.contains(key)) return dflt;
  return posint(j, key, ctx);
}

int64_t int_field(const ojson& j, const char* key, const char* ctx) {
  if (!j.contains(key) || !j[key].is_number_integer())
    throw ParseError(std::string(ctx) + ": missing integer field '" + key + "'");
  return j[key].get<int64_t>();
}

int device_ref(const ojson& v, const Cluster& c) {
  if (v.is_string()) {
    int i = c.device_index(v.get<std::string>());
    if (i < 0) throw ParseError("plan: unknown device id '" + v.get<std::string>() + "'");
    return i;
  }
  if (v.is_number_integer()) return v.get<int>();
  throw ParseError("plan: device reference must be an id string or index");
}

ojson id_list(const std::vector<int>& idxs, const Cluster& c) {
  ojson out = ojson::array();
  for (int i : idxs)
    out.push_back(i >= 0 && i < int(c.devices.size()) ? ojson(c.devices[i].id) : ojson(i));
  return out;
}

}  // namespace

int Cluster::device_index(const std::string& id) const {
  for (size_t i = 0; i < devices.size(); ++i)
    if (devices[i].id == id) return int(i);
  return -1;
}

double Cluster::max_peak() const {
  double m = 0;
  for (const auto& d : devices) m = std::max(m, d.peak_tflops);
  return m;
}

Cluster parse_cluster_doc(const std::string& text) {
  ojson j = parse_text(text, "cluster");
  if (!j.contains("machines") || !j["machines"].is_object())
    throw ParseError("cluster: missing 'machines' object");
  std::map<std::string, std::pair<double, double>> machines;  // name -> (bw, lat)
  for (auto& [name, mj] : j["machines"].items()) {
    const double bw = positive(mj, "intra_bandwidth_gbps", "machine") * 1e9;
    const double lat = nonneg(mj, "intra_latency_us", "machine") * 1e-6;
    machines[name] = {bw, lat};
  }
  if (!j.contains("devices") || !j["devices"].is_array() || j["devices"].empty())
    throw ParseError("cluster: missing or empty 'devices' array");
  Cluster c;
  std::set<std::string> seen;
  for (const auto& dj : j["devices"]) {
    Device d;
    if (!dj.contains("id") || !dj["id"].is_string())
      throw ParseError("device: missing string field 'id'");
    d.id = dj["id"].get<std::string>();
    if (!seen.insert(d.id).second) throw ParseError("device: duplicate id '" + d.id + "'");
    if (!dj.contains("machine") || !dj["machine"].is_string())
      throw ParseError("device '" + d.id + "': missing string field 'machine'");
    d.machine = dj["machine"].get<std::string>();
    if (!machines.count(d.machine))
      throw ParseError("device '" + d.id + "': unknown machine '" + d.machine + "'");
    d.memory_gib = positive(dj, "memory_gib", "device");
    d.peak_tflops = positive(dj, "peak_tflops", "device");
    if (dj.contains("rank")) d.rank = int(int_field(dj, "rank", "device"));
    if (dj.contains("sm_fraction")) {
      d.sm_fraction = positive(dj, "sm_fraction", "device");
      if (d.sm_fraction > 1.0) throw ParseError("device '" + d.id + "': sm_fraction > 1");
    }
    if (dj.contains("sm_count")) d.sm_count = int(posint(dj, "sm_count", "device"));
    c.devices.push_back(std::move(d));
  }
  if (!j.contains("inter") || !j["inter"].is_object())
    throw ParseError("cluster: missing 'inter' object");
  const double inter_bw = positive(j["inter"], "bandwidth_gbps", "inter") * 1e9;
  const double inter_lat = nonneg(j["inter"], "latency_us", "inter") * 1e-6;
  // per-pair overrides (json_io.cpp:120-147): unordered pairs, asymmetric
  // duplicates rejected with the reference's messages
  std::map<std::pair<int, int>, std::pair<double, double>> ov;
  if (j.contains("overrides")) {
    if (!j["overrides"].is_array()) throw ParseError("cluster: 'overrides' must be an array");
    for (const auto& oj : j["overrides"]) {
      if (!oj.contains("a") || !oj.contains("b") || !oj["a"].is_string() || !oj["b"].is_string())
        throw ParseError("override: needs string fields 'a' and 'b'");
      const std::string a = oj["a"].get<std::string>(), b = oj["b"].get<std::string>();
      const int ia = c.device_index(a), ib = c.device_index(b);
      if (ia < 0 || ib < 0) throw ParseError("override: unknown device '" + (ia < 0 ? a : b) + "'");
      if (ia == ib) throw ParseError("override: 'a' and 'b' must differ");
      const double bw = positive(oj, "bandwidth_gbps", "override") * 1e9;
      const double lat = nonneg(oj, "latency_us", "override") * 1e-6;
      const std::pair<int, int> key = std::minmax(ia, ib);
      auto it = ov.find(key);
      if (it != ov.end() && (it->second.first != bw || it->second.second != lat))
        throw ParseError("override: asymmetric bandwidth on pair '" + a + "'/'" + b + "'");
      ov[key] = {bw, lat};
    }
  }
  const size_t n = c.devices.size();
  c.bandwidth.assign(n, std::vector<double>(n, 0.0));
  c.latency.assign(n, std::vector<double>(n, 0.0));
  for (size_t a = 0; a < n; ++a)
    for (size_t b = a + 1; b < n; ++b) {
      double bw = inter_bw, lat = inter_lat;
      if (c.devices[a].machine == c.devices[b].machine) {
        bw = machines[c.devices[a].machine].first;
        lat = machines[c.devices[a].machine].second;
      }
      auto it = ov.find({int(a), int(b)});
      if (it != ov.end()) {
        bw = it->second.first;
        lat = it->second.second;
      }
      c.bandwidth[a][b] = c.bandwidth[b][a] = bw;
      c.latency[a][b] = c.latency[b][a] = lat;
    }
  return c;
}

Model parse_model_doc(const std::string& text) {
  ojson j = parse_text(text, "model");
  Model m;
  m.num_layers = posint(j, "num_layers", "model");
  m.hidden_dim = posint(j, "hidden_dim", "model");
  m.seq_len = posint(j, "seq_len", "model");
  m.bytes_per_element = posint(j, "bytes_per_element", "model");
  const int64_t H = m.hidden_dim;
  m.num_heads = opt_posint(j, "num_heads", H % 128 == 0 ? H / 128 : (H % 64 == 0 ? H / 64 : 1),
                           "model");
  // Llama rule: 8H/3 rounded up to a multiple of 256 (11008 / 13824 / 17920)
  int64_t f = (8 * H + 2) / 3;
  f = (f + 255) / 256 * 256;
  m.ffn_dim = opt_posint(j, "ffn_dim", f, "model");
  m.vocab_size = opt_posint(j, "vocab_size", 32000, "model");
  if (j.contains("rope_theta")) m.rope_theta = positive(j, "rope_theta", "model");
  if (j.contains("norm_eps")) m.norm_eps = positive(j, "norm_eps", "model");
  if (m.hidden_dim % m.num_heads != 0)
    throw InvalidArgument("model: hidden_dim not divisible by num_heads");
  if (m.head_dim() % 64 != 0 || m.head_dim() > 256)
    throw InvalidArgument("model: head_dim must be a multiple of 64 and <= 256");
  if (m.hidden_dim % 64 != 0) throw InvalidArgument("model: hidden_dim must be a multiple of 64");
  if (m.hidden_dim > 8192) throw InvalidArgument("model: hidden_dim must be <= 8192");
  if (m.ffn_dim % 64 != 0) throw InvalidArgument("model: ffn_dim must be a multiple of 64");
  if (m.vocab_size % 64 != 0) throw InvalidArgument("model: vocab_size must be a multiple of 64");
  if (m.vocab_size > 65536) throw InvalidArgument("model: vocab_size must be <= 65536");
  if (m.seq_len % 128 != 0) throw InvalidArgument("model: seq_len must be a multiple of 128");
  return m;
}

Plan parse_plan_doc(const std::string& text, const Cluster& c, bool* had_dp_groups) {
  ojson j = parse_text(text, "plan");
  // CLI artifact: {"manifest": {...}, "plan": {...}} (hexplan_cli.cpp:217-218)
  if (j.is_object() && j.contains("plan") && j["plan"].is_object()) j = j["plan"];
  if (!j.is_object()) throw ParseError("plan: expected an object");
  Plan p;
  p.global_batch = int_field(j, "global_batch", "plan");
  if (!j.contains("pipelines") || !j["pipelines"].is_array())
    throw ParseError("plan: missing 'pipelines' array");
  for (const auto& jp : j["pipelines"]) {
    Pipeline pp;
    pp.batch = int_field(jp, "batch", "pipeline");
    pp.micro_batch = int_field(jp, "micro_batch", "pipeline");
    if (!jp.contains("stages") || !jp["stages"].is_array())
      throw ParseError("pipeline: missing 'stages' array");
    for (const auto& js : jp["stages"]) {
      Stage st;
      if (!js.contains("devices") || !js["devices"].is_array())
        throw ParseError("stage: missing 'devices' array");
      for (const auto& d : js["devices"]) st.devices.push_back(device_ref(d, c));
      st.tp = int(int_field(js, "tp", "stage"));
      st.layer_start = int(int_field(js, "layer_start", "stage"));
      st.layer_count = int(int_field(js, "layer_count", "stage"));
      if (js.contains("tp_widths")) {
        if (!js["tp_widths"].is_array()) throw ParseError("stage: 'tp_widths' must be an array");
        for (const auto& w : js["tp_widths"]) {
          if (!w.is_number_integer() || w.get<int64_t>() <= 0)
            throw ParseError("stage: 'tp_widths' entries must be positive integers");
          st.tp_widths.push_back(w.get<int64_t>());
        }
      }
      pp.stages.push_back(std::move(st));
    }
    p.pipelines.push_back(std::move(pp));
  }
  *had_dp_groups = j.contains("dp_groups");
  if (*had_dp_groups) {
    if (!j["dp_groups"].is_array()) throw ParseError("plan: 'dp_groups' must be an array");
    for (const auto& jg : j["dp_groups"]) {
      DpGroup g;
      g.layer = int(int_field(jg, "layer", "dp_group"));
      if (!jg.contains("members") || !jg["members"].is_array())
        throw ParseError("dp_group: missing 'members' array");
      for (const auto& d : jg["members"]) g.members.push_back(device_ref(d, c));
      p.dp_groups.push_back(std::move(g));
    }
  }
  return p;
}

void build_dp_groups(Plan& plan, const Model& m) {
  plan.dp_groups.assign(size_t(m.num_layers), DpGroup{});
  for (int64_t l = 0; l < m.num_layers; ++l) plan.dp_groups[size_t(l)].layer = int(l);
  for (const auto& p : plan.pipelines)
    for (const auto& st : p.stages) {
      if (st.devices.empty()) continue;  // validate_plan rejects it afterwards
      for (int l = st.layer_start; l < st.layer_start + st.layer_count; ++l)
        if (l >= 0 && l < m.num_layers) plan.dp_groups[size_t(l)].members.push_back(st.devices[0]);
    }
}

void validate_plan(const Plan& plan, const Model& m, const Cluster& c) {
  if (plan.pipelines.empty()) throw InvalidArgument("plan has no pipelines");
  if (plan.global_batch < 1) throw InvalidArgument("plan has no batch");
  std::vector<char> used(c.devices.size(), 0);
  int64_t batch_sum = 0;
  for (const auto& p : plan.pipelines) {
    if (p.stages.empty()) throw InvalidArgument("pipeline has no stages");
    if (p.micro_batch < 1 || p.batch < p.micro_batch)
      throw InvalidArgument("pipeline batch smaller than its micro batch");
    if (p.batch % p.micro_batch != 0)
      throw InvalidArgument("pipeline batch not a micro batch multiple");
    batch_sum += p.batch;
    int next = 0;
    for (const auto& st : p.stages) {
      if (st.devices.empty()) throw InvalidArgument("stage has no devices");
      if (st.tp != int(st.devices.size()))
        throw InvalidArgument("stage tp degree does not match its device count");
      if (st.layer_count < 1) throw InvalidArgument("stage holds no layers");
      if (st.layer_start != next) throw InvalidArgument("stages do not tile the layer range");
      next += st.layer_count;
      for (int d : st.devices) {
        if (d < 0 || d >= int(c.devices.size()))
          throw InvalidArgument("stage references an unknown device");
        if (used[size_t(d)]) throw InvalidArgument("device appears in two stages");
        used[size_t(d)] = 1;
      }
    }
    if (next != m.num_layers) throw InvalidArgument("pipeline does not cover all layers");
  }
  if (batch_sum != plan.global_batch)
    throw InvalidArgument("pipeline batches do not sum to the global batch");
  if (plan.dp_groups.size() != size_t(m.num_layers))
    throw InvalidArgument("dp groups do not cover all layers");
  for (size_t l = 0; l < plan.dp_groups.size(); ++l) {
    if (plan.dp_groups[l].layer != int(l))
      throw InvalidArgument("dp group layer index out of order");
    if (plan.dp_groups[l].members.size() != plan.pipelines.size())
      throw InvalidArgument("dp group missing a pipeline replica");
  }
}

std::vector<int64_t> largest_remainder(int64_t units, const std::vector<int64_t>& w) {
  int64_t W = 0;
  for (int64_t x : w) W += x;
  std::vector<int64_t> out(w.size(), 0);
  if (W <= 0) return out;
  std::vector<std::pair<int64_t, size_t>> rem;  // (remainder, index)
  int64_t assigned = 0;
  for (size_t i = 0; i < w.size(); ++i) {
    __int128 q = (__int128)units * w[i];
    out[i] = int64_t(q / W);
    rem.push_back({int64_t(q % W), i});
    assigned += out[i];
  }
  std::stable_sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
    if (a.first != b.first) return a.first > b.first;
    return a.second < b.second;
  });
  for (int64_t k = 0; k < units - assigned; ++k) out[rem[size_t(k)].second] += 1;
  return out;
}

std::string serialize_plan(const Plan& plan, const Cluster& c) {
  ojson j;
  j["global_batch"] = plan.global_batch;
  j["pipelines"] = ojson::array();
  for (const auto& p : plan.pipelines) {
    ojson jp;
    jp["batch"] = p.batch;
    jp["micro_batch"] = p.micro_batch;
    jp["num_micro_batches"] = p.num_micro_batches();
    jp["stages"] = ojson::array();
    for (const auto& s : p.stages) {
      ojson js;
      js["devices"] = id_list(s.devices, c);
      js["tp"] = s.tp;
      js["layer_start"] = s.layer_start;
      js["layer_count"] = s.layer_count;
      jp["stages"].push_back(std::move(js));
    }
    j["pipelines"].push_back(std::move(jp));
  }
  j["dp_groups"] = ojson::array();
  for (const auto& g : plan.dp_groups) {
    ojson jg;
    jg["layer"] = g.layer;
    jg["members"] = id_list(g.members, c);
    j["dp_groups"].push_back(std::move(jg));
  }
  return j.dump(2) + "\n";
}

namespace {

std::vector<TensorSpec> make_catalogue(const Model& m) {
  std::vector<TensorSpec> t;
  const int64_t H = m.hidden_dim, F = m.ffn_dim, V = m.vocab_size;
  t.push_back({"embed", -1, kEmbed, V, H, true});
  for (int l = 0; l < int(m.num_layers); ++l) {
    std::string p = "layers." + std::to_string(l) + ".";
    t.push_back({p + "attn_norm", l, kAttnNorm, 1, H, false});
    t.push_back({p + "wqkv", l, kWqkv, 3 * H, H, true});
    t.push_back({p + "wo", l, kWo, H, H, true});
    t.push_back({p + "mlp_norm", l, kMlpNorm, 1, H, false});
    t.push_back({p + "wgu", l, kWgu, 2 * F, H, true});
    t.push_back({p + "wdown", l, kWdown, F, H, true});
  }
  t.push_back({"final_norm", -1, kFinalNorm, 1, H, false});
  t.push_back({"lm_head", -1, kLmHead, V, H, true});
  return t;
}

// row range of tensor `s` held by `r` (rows == 0: not held)
void rows_of(const TensorSpec& s, const RankRole& r, const Model& m, int64_t* row0,
             int64_t* rows, int* mult) {
  *row0 = 0;
  *rows = 0;
  *mult = 1;
  if (!r.active) return;
  const int64_t d = m.head_dim();
  bool held;
  if (s.layer >= 0)
    held = s.layer >= r.layer_start && s.layer < r.layer_start + r.layer_count;
  else if (s.id == kEmbed)
    held = r.first_stage;
  else
    held = r.last_stage;
  if (!held) return;
  switch (s.id) {
    case kEmbed:
    case kAttnNorm:
    case kMlpNorm:
    case kFinalNorm:
      *rows = s.global_rows;
      *mult = r.tp;
      return;
    case kWqkv:
      *row0 = 3 * d * r.heads.begin;
      *rows = 3 * d * r.heads.size();
      return;
    case kWo:
      *row0 = d * r.heads.begin;
      *rows = d * r.heads.size();
      return;
    case kWgu:
      *row0 = 128 * r.ffn_chunks.begin;
      *rows = 128 * r.ffn_chunks.size();
      return;
    case kWdown:
      *row0 = 64 * r.ffn_chunks.begin;
      *rows = 64 * r.ffn_chunks.size();
      return;
    case kLmHead:
      *row0 = 64 * r.vocab_chunks.begin;
      *rows = 64 * r.vocab_chunks.size();
      return;
  }
}

}  // namespace

int sync_group(const TensorSpec& t) {
  if (t.layer >= 0) return t.layer;
  return t.id == kEmbed ? kGroupEmbed : kGroupHead;
}

namespace {

int intern_set(std::vector<std::vector<int>>& sets, std::map<std::vector<int>, int>& idx,
               std::vector<int> s) {
  std::sort(s.begin(), s.end());
  auto it = idx.find(s);
  if (it != idx.end()) return it->second;
  sets.push_back(s);
  idx[s] = int(sets.size()) - 1;
  return int(sets.size()) - 1;
}

}  // namespace

Layout build_layout(const std::string& cluster_json, const std::string& model_json,
                    const std::string& plan_json) {
  Layout L;
  L.cluster = parse_cluster_doc(cluster_json);
  L.model = parse_model_doc(model_json);
  bool had = false;
  L.plan = parse_plan_doc(plan_json, L.cluster, &had);
  if (!had) build_dp_groups(L.plan, L.model);
  validate_plan(L.plan, L.model, L.cluster);
  const Model& m = L.model;
  const Cluster& c = L.cluster;

  // world ranks: "rank" extension or document order; must be a bijection
  const int n = int(c.devices.size());
  L.world_size = n;
  L.rank_of_device.assign(size_t(n), -1);
  L.device_of_rank.assign(size_t(n), -1);
  for (int i = 0; i < n; ++i) {
    int r = c.devices[size_t(i)].rank >= 0 ? c.devices[size_t(i)].rank : i;
    if (r >= n) throw InvalidArgument("device rank out of range");
    if (L.device_of_rank[size_t(r)] >= 0) throw InvalidArgument("two devices share a rank");
    L.rank_of_device[size_t(i)] = r;
    L.device_of_rank[size_t(r)] = i;
  }

  L.tensors = make_catalogue(m);
  L.roles.assign(size_t(n), RankRole{});
  // emulated tier: the device's share of a full B200 (2250 TFLOPS dense BF16,
  // the c_d the probe clusters use), capped at 1
  constexpr double kB200Peak = 2250.0;
  for (int r = 0; r < n; ++r) {
    RankRole& role = L.roles[size_t(r)];
    role.device = L.device_of_rank[size_t(r)];
    const Device& dv = c.devices[size_t(role.device)];
    role.sm_fraction =
        dv.sm_fraction > 0 ? dv.sm_fraction : std::min(1.0, dv.peak_tflops / kB200Peak);
    role.sm_count = dv.sm_count;
  }

  int64_t sample_off = 0;
  for (int pi = 0; pi < int(L.plan.pipelines.size()); ++pi) {
    const Pipeline& p = L.plan.pipelines[size_t(pi)];
    for (int sj = 0; sj < int(p.stages.size()); ++sj) {
      const Stage& st = p.stages[size_t(sj)];
      std::vector<int64_t> w = st.tp_widths;
      if (w.empty()) w.assign(size_t(st.tp), 1);
      if (int(w.size()) != st.tp)
        throw InvalidArgument("stage tp_widths length does not match its device count");
      auto heads = largest_remainder(m.num_heads, w);
      auto ffn = largest_remainder(m.ffn_dim / 64, w);
      auto voc = largest_remainder(m.vocab_size / 64, w);
      int64_t h0 = 0, f0 = 0, v0 = 0;
      std::vector<int> group;
      for (int d : st.devices) group.push_back(L.rank_of_device[size_t(d)]);
      for (int t = 0; t < st.tp; ++t) {
        if (heads[size_t(t)] < 1) throw InvalidArgument("tp shard holds no attention heads");
        if (ffn[size_t(t)] < 1) throw InvalidArgument("tp shard holds no ffn columns");
        if (voc[size_t(t)] < 1) throw InvalidArgument("tp shard holds no vocab rows");
        RankRole& role = L.roles[size_t(group[size_t(t)])];
        role.active = true;
        role.pipeline = pi;
        role.stage = sj;
        role.stage_count = int(p.stages.size());
        role.tp_index = t;
        role.tp = st.tp;
        role.layer_start = st.layer_start;
        role.layer_count = st.layer_count;
        role.first_stage = sj == 0;
        role.last_stage = sj + 1 == int(p.stages.size());
        role.heads = {h0, h0 + heads[size_t(t)]};
        role.ffn_chunks = {f0, f0 + ffn[size_t(t)]};
        role.vocab_chunks = {v0, v0 + voc[size_t(t)]};
        h0 += heads[size_t(t)];
        f0 += ffn[size_t(t)];
        v0 += voc[size_t(t)];
        role.sample0 = sample_off;
        role.batch = p.batch;
        role.micro_batch = p.micro_batch;
        role.n_mb = p.num_micro_batches();
        role.tp_group = group;
        role.dp_weight = double(p.batch) / double(L.plan.global_batch);
        // PP peers: receiver t takes from sender (t mod tp_sender)
        if (sj > 0) {
          const Stage& prev = p.stages[size_t(sj - 1)];
          role.fwd_recv_from = L.rank_of_device[size_t(prev.devices[size_t(t % prev.tp)])];
          for (int u = 0; u < prev.tp; ++u)
            if (u % st.tp == t) role.bwd_send_to.push_back(L.rank_of_device[size_t(prev.devices[size_t(u)])]);
        }
        if (sj + 1 < int(p.stages.size())) {
          const Stage& next = p.stages[size_t(sj + 1)];
          role.bwd_recv_from = L.rank_of_device[size_t(next.devices[size_t(t % next.tp)])];
          for (int u = 0; u < next.tp; ++u)
            if (u % st.tp == t) role.fwd_send_to.push_back(L.rank_of_device[size_t(next.devices[size_t(u)])]);
        }
      }
    }
    sample_off += p.batch;
  }

  // per-rank tensor shards in flat-buffer order
  for (int r = 0; r < n; ++r) {
    RankRole& role = L.roles[size_t(r)];
    int64_t off = 0;
    for (int s = 0; s < int(L.tensors.size()); ++s) {
      int64_t row0, rows;
      int mult;
      rows_of(L.tensors[size_t(s)], role, m, &row0, &rows, &mult);
      if (rows == 0) continue;
      RankTensor rt;
      rt.spec = s;
      rt.row0 = row0;
      rt.rows = rows;
      rt.offset = off;
      rt.multiplicity = mult;
      role.tensors.push_back(rt);
      off += rows * L.tensors[size_t(s)].cols;
    }
    role.param_count = off;
  }

  // communicator sets: TP groups + chunk-matched DP participant sets
  std::map<std::vector<int>, int> set_idx;
  L.tp_comm.assign(size_t(n), -1);
  for (int r = 0; r < n; ++r) {
    const RankRole& role = L.roles[size_t(r)];
    if (role.active && role.tp > 1) L.tp_comm[size_t(r)] = intern_set(L.comm_sets, set_idx, role.tp_group);
  }
  L.dp_buckets.assign(size_t(n), {});
  L.dp_scales.assign(size_t(n), {});
  for (int r = 0; r < n; ++r) {
    const RankRole& role = L.roles[size_t(r)];
    for (const auto& rt : role.tensors)
      L.dp_scales[size_t(r)].push_back({rt.offset, rt.rows * L.tensors[size_t(rt.spec)].cols,
                                        float(role.dp_weight / double(rt.multiplicity))});
  }
  // holders per tensor
  struct Holder { int rank; int64_t b, e, local; };
  struct Seg { std::vector<int> ranks; std::vector<int64_t> local; int64_t len; int group; };
  std::vector<Seg> segs;
  for (int s = 0; s < int(L.tensors.size()); ++s) {
    const int64_t cols = L.tensors[size_t(s)].cols;
    const int group = sync_group(L.tensors[size_t(s)]);
    std::vector<Holder> hs;
    std::vector<int64_t> cuts;
    for (int r = 0; r < n; ++r)
      for (const auto& rt : L.roles[size_t(r)].tensors)
        if (rt.spec == s) {
          hs.push_back({r, rt.row0 * cols, (rt.row0 + rt.rows) * cols, rt.offset});
          cuts.push_back(rt.row0 * cols);
          cuts.push_back((rt.row0 + rt.rows) * cols);
        }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    for (size_t k = 0; k + 1 < cuts.size(); ++k) {
      Seg sg;
      sg.len = cuts[k + 1] - cuts[k];
      sg.group = group;
      for (const auto& h : hs)
        if (h.b <= cuts[k] && cuts[k + 1] <= h.e) {
          sg.ranks.push_back(h.rank);
          sg.local.push_back(h.local + (cuts[k] - h.b));
        }
      if (sg.ranks.size() >= 2 && sg.len > 0) segs.push_back(std::move(sg));
    }
  }
  // merge consecutive segments that are contiguous on every participant
  std::vector<Seg> merged;
  for (auto& sg : segs) {
    if (!merged.empty()) {
      Seg& b = merged.back();
      // buckets never span two sync groups (layer / embedding / head), so each
      // becomes reducible as soon as its group's backward of the last
      // micro-batch is done
      bool ok = b.ranks == sg.ranks && b.group == sg.group;
      for (size_t i = 0; ok && i < sg.ranks.size(); ++i) ok = b.local[i] + b.len == sg.local[i];
      if (ok) {
        b.len += sg.len;
        continue;
      }
    }
    merged.push_back(sg);
  }
  for (const auto& sg : merged) {
    int ci = intern_set(L.comm_sets, set_idx, sg.ranks);
    for (size_t i = 0; i < sg.ranks.size(); ++i)
      L.dp_buckets[size_t(sg.ranks[i])].push_back({ci, sg.local[i], sg.len, sg.group});
  }
  return L;
}

std::string layout_json(const Layout& L) {
  ojson j;
  j["world_size"] = L.world_size;
  j["model"] = {{"num_layers", L.model.num_layers}, {"hidden_dim", L.model.hidden_dim},
                {"seq_len", L.model.seq_len}, {"num_heads", L.model.num_heads},
                {"head_dim", L.model.head_dim()}, {"ffn_dim", L.model.ffn_dim},
                {"vocab_size", L.model.vocab_size}, {"rope_theta", L.model.rope_theta},
                {"norm_eps", L.model.norm_eps}};
  j["num_micro_batches"] = ojson::array();
  for (const auto& p : L.plan.pipelines) j["num_micro_batches"].push_back(p.num_micro_batches());
  j["dp_groups"] = ojson::array();
  for (const auto& g : L.plan.dp_groups)
    j["dp_groups"].push_back({{"layer", g.layer}, {"members", id_list(g.members, L.cluster)}});
  j["comm_sets"] = L.comm_sets;
  j["ranks"] = ojson::array();
  for (int r = 0; r < L.world_size; ++r) {
    const RankRole& ro = L.roles[size_t(r)];
    ojson jr;
    jr["rank"] = r;
    jr["device"] = L.cluster.devices[size_t(ro.device)].id;
    jr["active"] = ro.active;
    jr["sm_fraction"] = ro.sm_fraction;
    if (ro.active) {
      jr["pipeline"] = ro.pipeline;
      jr["stage"] = ro.stage;
      jr["tp_index"] = ro.tp_index;
      jr["tp"] = ro.tp;
      jr["layers"] = {ro.layer_start, ro.layer_start + ro.layer_count};
      jr["heads"] = {ro.heads.begin, ro.heads.end};
      jr["ffn_cols"] = {64 * ro.ffn_chunks.begin, 64 * ro.ffn_chunks.end};
      jr["vocab_rows"] = {64 * ro.vocab_chunks.begin, 64 * ro.vocab_chunks.end};
      jr["samples"] = {ro.sample0, ro.sample0 + ro.batch};
      jr["micro_batch"] = ro.micro_batch;
      jr["num_micro_batches"] = ro.n_mb;
      jr["tp_group"] = ro.tp_group;
      jr["tp_comm"] = L.tp_comm[size_t(r)];
      jr["fwd_recv_from"] = ro.fwd_recv_from;
      jr["bwd_recv_from"] = ro.bwd_recv_from;
      jr["fwd_send_to"] = ro.fwd_send_to;
      jr["bwd_send_to"] = ro.bwd_send_to;
      jr["dp_weight"] = ro.dp_weight;
      jr["param_count"] = ro.param_count;
      ojson ts = ojson::array();
      for (const auto& rt : ro.tensors)
        ts.push_back({{"name", L.tensors[size_t(rt.spec)].name}, {"row0", rt.row0},
                      {"rows", rt.rows}, {"cols", L.tensors[size_t(rt.spec)].cols},
                      {"offset", rt.offset}, {"multiplicity", rt.multiplicity}});
      jr["tensors"] = ts;
      ojson bk = ojson::array();
      for (const auto& b : L.dp_buckets[size_t(r)])
        bk.push_back({{"comm", b.comm}, {"offset", b.offset}, {"count", b.count},
                      {"group", b.group}});
      jr["dp_buckets"] = bk;
    }
    j["ranks"].push_back(std::move(jr));
  }
  return j.dump();
}

}  // namespace hexexec
