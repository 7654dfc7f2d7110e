// Canonical trace JSON (ref src/trace.cpp:159-315) and the three synthetic
// trace generators (ref src/trace.cpp:317-476).  Both are harness-side: they
// let the bundled fixtures (data/*.json) be reproduced byte-for-byte and let
// the B200 runtime export the traces it plans with in the reference format.
#include <random>

#include <nlohmann/json.hpp>

#include "deltasim/deltasim.hpp"

namespace deltasim {

using ojson = nlohmann::ordered_json;

namespace {

void only_keys(const ojson& obj, std::initializer_list<const char*> allowed,
               const std::string& where) {
  for (auto it = obj.begin(); it != obj.end(); ++it) {
    bool known = false;
    for (const char* k : allowed) known |= it.key() == k;
    if (!known) throw SchemaError(where + ": unknown field '" + it.key() + "'");
  }
}

const ojson& field(const ojson& obj, const char* key, const std::string& where) {
  auto it = obj.find(key);
  if (it == obj.end()) throw SchemaError(where + ": missing field '" + key + "'");
  return *it;
}

std::uint64_t u64_of(const ojson& j, const char* key, const std::string& where) {
  if (!j.is_number_unsigned())
    throw SchemaError(where + ": field '" + key + "' must be an unsigned integer");
  return j.get<std::uint64_t>();
}

bool bool_of(const ojson& j, const char* key, const std::string& where) {
  if (!j.is_boolean()) throw SchemaError(where + ": field '" + key + "' must be a boolean");
  return j.get<bool>();
}

std::string str_of(const ojson& j, const char* key, const std::string& where) {
  if (!j.is_string()) throw SchemaError(where + ": field '" + key + "' must be a string");
  return j.get<std::string>();
}

}  // namespace

Trace parse_trace(const std::string& text) {
  ojson root = ojson::parse(text, nullptr, false);
  if (root.is_discarded()) throw SchemaError("document is not well-formed JSON");
  if (!root.is_object()) throw SchemaError("top level must be an object");
  const std::string top = "top level";
  only_keys(root, {"name", "nodes", "schedule"}, top);
  Trace t;
  t.name = str_of(field(root, "name", top), "name", top);

  const ojson& nodes = field(root, "nodes", top);
  if (!nodes.is_array()) throw SchemaError("'nodes' must be an array");
  t.nodes.reserve(nodes.size());
  for (std::size_t i = 0; i < nodes.size(); ++i) {
    const std::string w = "nodes[" + std::to_string(i) + "]";
    const ojson& jn = nodes[i];
    if (!jn.is_object()) throw SchemaError(w + ": must be an object");
    only_keys(jn, {"id", "name", "compute_cost_us", "output_bytes", "parents",
                   "uncomputable", "evict_pinned", "offload_pinned"},
              w);
    OpNode n;
    n.id = u64_of(field(jn, "id", w), "id", w);
    n.name = str_of(field(jn, "name", w), "name", w);
    n.compute_cost_us = u64_of(field(jn, "compute_cost_us", w), "compute_cost_us", w);
    n.output_bytes = u64_of(field(jn, "output_bytes", w), "output_bytes", w);
    const ojson& ps = field(jn, "parents", w);
    if (!ps.is_array()) throw SchemaError(w + ": field 'parents' must be an array");
    for (const ojson& p : ps) n.parents.push_back(u64_of(p, "parents", w));
    n.uncomputable = bool_of(field(jn, "uncomputable", w), "uncomputable", w);
    n.evict_pinned = bool_of(field(jn, "evict_pinned", w), "evict_pinned", w);
    n.offload_pinned = bool_of(field(jn, "offload_pinned", w), "offload_pinned", w);
    t.nodes.push_back(std::move(n));
  }

  const ojson& sched = field(root, "schedule", top);
  if (!sched.is_array()) throw SchemaError("'schedule' must be an array");
  t.schedule.reserve(sched.size());
  for (std::size_t i = 0; i < sched.size(); ++i) {
    const std::string w = "schedule[" + std::to_string(i) + "]";
    const ojson& je = sched[i];
    if (!je.is_object()) throw SchemaError(w + ": must be an object");
    only_keys(je, {"node", "phase", "kind"}, w);
    AccessEvent ev;
    ev.node = u64_of(field(je, "node", w), "node", w);
    const std::string ph = str_of(field(je, "phase", w), "phase", w);
    if (ph == "F")
      ev.phase = Phase::Forward;
    else if (ph == "B")
      ev.phase = Phase::Backward;
    else
      throw SchemaError(w + ": field 'phase' must be \"F\" or \"B\"");
    const std::string kd = str_of(field(je, "kind", w), "kind", w);
    if (kd == "P")
      ev.kind = AccessKind::Produce;
    else if (kd == "U")
      ev.kind = AccessKind::Use;
    else
      throw SchemaError(w + ": field 'kind' must be \"P\" or \"U\"");
    t.schedule.push_back(ev);
  }
  for (const TraceViolation& v : validate_trace(t))
    if (v.severity == Severity::Error) throw ValidationErrorEx(v.message);
  return t;
}

std::string serialize_trace(const Trace& t) {
  ojson root;
  root["name"] = t.name;
  ojson nodes = ojson::array();
  for (const OpNode& n : t.nodes) {
    ojson j;
    j["id"] = n.id;
    j["name"] = n.name;
    j["compute_cost_us"] = n.compute_cost_us;
    j["output_bytes"] = n.output_bytes;
    j["parents"] = n.parents;
    j["uncomputable"] = n.uncomputable;
    j["evict_pinned"] = n.evict_pinned;
    j["offload_pinned"] = n.offload_pinned;
    nodes.push_back(std::move(j));
  }
  root["nodes"] = std::move(nodes);
  ojson sched = ojson::array();
  for (const AccessEvent& e : t.schedule) {
    ojson j;
    j["node"] = e.node;
    j["phase"] = e.phase == Phase::Forward ? "F" : "B";
    j["kind"] = e.kind == AccessKind::Produce ? "P" : "U";
    sched.push_back(std::move(j));
  }
  root["schedule"] = std::move(sched);
  return root.dump();
}

// ---------------------------------------------------------------------------
// Generators.  Jitter: seed 0 disables; otherwise v * (90 + raw % 21) / 100,
// floored at 1, drawing one raw mt19937_64 output per non-zero value.

namespace {

struct Builder {
  Trace t;
  std::uint64_t seed;
  std::mt19937_64 rng;
  explicit Builder(std::string name, std::uint64_t s) : seed(s), rng(s) {
    t.name = std::move(name);
  }
  std::uint64_t jit(std::uint64_t v) {
    if (seed == 0 || v == 0) return v;
    std::uint64_t scaled = v * (90 + rng() % 21) / 100;
    return scaled ? scaled : 1;
  }
  NodeId add(std::string name, MicroDur cost, Bytes bytes,
             std::vector<NodeId> parents, bool input) {
    OpNode n;
    n.id = t.nodes.size();
    n.name = std::move(name);
    n.compute_cost_us = jit(cost);
    n.output_bytes = jit(bytes);
    n.parents = std::move(parents);
    n.uncomputable = input;
    n.evict_pinned = input;
    t.nodes.push_back(std::move(n));
    return t.nodes.back().id;
  }
  // Forward produces in declaration order; backward uses in reverse.
  void forward_then_reverse() {
    for (const OpNode& n : t.nodes) t.schedule.push_back({n.id, Phase::Forward, AccessKind::Produce});
    for (std::size_t i = t.nodes.size(); i-- > 0;)
      t.schedule.push_back({t.nodes[i].id, Phase::Backward, AccessKind::Use});
  }
};

}  // namespace

Trace gen_linear_chain(std::size_t n, Bytes bytes_per, MicroDur cost_per,
                       std::uint64_t seed) {
  if (n == 0) throw ArgumentError("gen_linear_chain: n must be >= 1");
  Builder b("linear" + std::to_string(n), seed);
  for (std::size_t i = 0; i < n; ++i) {
    // cost is jittered before bytes for every node, including the input
    OpNode node;
    node.id = i;
    node.name = i == 0 ? "Input" : "LinearForward" + std::to_string(i);
    node.compute_cost_us = b.jit(cost_per);
    node.output_bytes = b.jit(bytes_per);
    if (i == 0) {
      node.uncomputable = node.evict_pinned = true;
    } else {
      node.parents.push_back(i - 1);
    }
    b.t.nodes.push_back(std::move(node));
  }
  for (std::size_t i = 0; i < n; ++i) b.t.schedule.push_back({i, Phase::Forward, AccessKind::Produce});
  for (std::size_t i = n; i-- > 0;) {  // layer i's gradient reads i and i-1
    b.t.schedule.push_back({i, Phase::Backward, AccessKind::Use});
    if (i >= 1) b.t.schedule.push_back({i - 1, Phase::Backward, AccessKind::Use});
  }
  return std::move(b.t);
}

Trace gen_resnet_like(std::size_t blocks, Bytes branch_bytes,
                      std::uint64_t seed) {
  if (blocks == 0) throw ArgumentError("gen_resnet_like: blocks must be >= 1");
  Builder b("resnet" + std::to_string(blocks), seed);
  const Bytes small = branch_bytes / 4 == 0 ? 1 : branch_bytes / 4;
  NodeId cur = b.add("Input", 0, small, {}, true);
  for (std::size_t k = 0; k < blocks; ++k) {
    const std::string sfx = "_" + std::to_string(k);
    NodeId conv = b.add("ConvForward" + sfx, 200, 2 * branch_bytes, {cur}, false);
    NodeId bn = b.add("BNForward" + sfx, 5, branch_bytes, {conv}, false);
    NodeId relu = b.add("ReLUForward" + sfx, 3, branch_bytes, {bn}, false);
    cur = b.add("AddForward" + sfx, 4, small, {cur, relu}, false);
  }
  b.forward_then_reverse();
  return std::move(b.t);
}

Trace gen_transformer_like(std::size_t layers, Bytes hidden_bytes,
                           std::uint64_t seed) {
  if (layers == 0) throw ArgumentError("gen_transformer_like: layers must be >= 1");
  Builder b("transformer" + std::to_string(layers), seed);
  const Bytes h = hidden_bytes;
  NodeId cur = b.add("Embedding", 0, h, {}, true);
  for (std::size_t l = 0; l < layers; ++l) {
    const std::string s = "_" + std::to_string(l);
    NodeId ln1 = b.add("LayerNorm1" + s, 4, h, {cur}, false);
    NodeId qkv = b.add("QKVProj" + s, 120, 3 * h, {ln1}, false);
    NodeId attn = b.add("Attention" + s, 180, h, {qkv}, false);
    NodeId proj = b.add("OutProj" + s, 60, h, {attn}, false);
    NodeId add1 = b.add("AddResid1" + s, 4, h, {cur, proj}, false);
    NodeId ln2 = b.add("LayerNorm2" + s, 4, h, {add1}, false);
    NodeId up = b.add("MlpUp" + s, 150, 4 * h, {ln2}, false);
    NodeId down = b.add("MlpDown" + s, 150, h, {up}, false);
    cur = b.add("AddResid2" + s, 4, h, {add1, down}, false);
  }
  b.forward_then_reverse();
  return std::move(b.t);
}

}  // namespace deltasim
