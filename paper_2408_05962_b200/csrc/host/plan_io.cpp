// Plan persistence: hiercoll-plan-v1 (a lowered plan) and
// hiercoll-pipelined-v1 (the same plus pipeline depth and slot count).
// Field names and their order are the reference's (factorize.cpp:680-788,
// pipeline.cpp:147-172) so the text is byte-identical and plans can be
// diffed against the reference's or fed to it.
#include "planning.hpp"

namespace hiccl {

namespace {

const char* op_name(const P2PTransfer& t) {
  if (!t.reduce) return "copy";
  return t.op == ReduceOp::max ? "max" : "sum";
}

json::Value transfer_to_json(const P2PTransfer& t) {
  json::Value o = json::Value::Obj();
  const std::pair<const char*, int64_t> head[] = {
      {"id", t.id},       {"stage", t.stage}, {"level", t.level}, {"stripe", t.stripe},
      {"channel", t.channel}, {"slot", t.slot}, {"src", t.src},   {"dst", t.dst}};
  for (const auto& [k, v] : head) o.set(k, json::Value::Int(v));
  o.set("src_buffer", json::Value::Str(t.src_buffer));
  o.set("src_offset", json::Value::Int(t.src_offset));
  o.set("dst_buffer", json::Value::Str(t.dst_buffer));
  o.set("dst_offset", json::Value::Int(t.dst_offset));
  o.set("count", json::Value::Int(t.count));
  o.set("op", json::Value::Str(op_name(t)));
  o.set("step", json::Value::Int(t.step));
  o.set("deps", json::Value::IntArr(t.deps));
  return o;
}

P2PTransfer transfer_from_json(const json::Value& o) {
  P2PTransfer t;
  auto i32 = [&](const char* k) { return (int)o.at(k).as_int(); };
  t.id = i32("id");
  t.stage = i32("stage");
  t.level = i32("level");
  t.stripe = i32("stripe");
  t.channel = (int)o.int_or("channel", 0);
  t.slot = (int)o.int_or("slot", t.stage);
  t.src = i32("src");
  t.dst = i32("dst");
  t.src_buffer = o.at("src_buffer").as_str();
  t.src_offset = o.at("src_offset").as_int();
  t.dst_buffer = o.at("dst_buffer").as_str();
  t.dst_offset = o.at("dst_offset").as_int();
  t.count = o.at("count").as_int();
  const std::string& op = o.at("op").as_str();
  t.reduce = op != "copy";
  if (t.reduce) t.op = reduce_op_from_string(op);
  t.step = (int)o.int_or("step", 0);
  t.deps = o.at("deps").as_int_vec<int>();
  return t;
}

json::Value parse_as(const std::string& text, const char* format) {
  json::Value doc = json::parse(text);
  if (doc.type != json::Value::Type::object || doc.str_or("format", "") != format)
    throw Error(ErrorCode::ParseError, std::string("expected a ") + format + " document");
  return doc;
}

}  // namespace

json::Value staged_plan_json(const StagedPlan& p) {
  json::Value doc = json::Value::Obj();
  doc.set("format", json::Value::Str("hiercoll-plan-v1"));
  doc.set("world_size", json::Value::Int(p.world_size));
  doc.set("element_size", json::Value::Int(p.element_size));
  doc.set("stripe", json::Value::Int(p.stripe));
  doc.set("ring", json::Value::Int(p.ring));
  doc.set("num_stages", json::Value::Int(p.num_stages));
  doc.set("source_program_id", json::Value::Str(p.source_program_id));
  doc.set("buffers", buffers_to_json(p.buffers));
  json::Value fences = json::Value::Arr();
  for (const auto& f : p.fences) {
    json::Value o = json::Value::Obj();
    o.set("stage", json::Value::Int(f.stage));
    o.set("aligned", json::Value::Bool(f.aligned));
    fences.push(std::move(o));
  }
  doc.set("fences", std::move(fences));
  json::Value ts = json::Value::Arr();
  ts.arr.reserve(p.transfers.size());
  for (const auto& t : p.transfers) ts.push(transfer_to_json(t));
  doc.set("transfers", std::move(ts));
  return doc;
}

StagedPlan staged_plan_from(const json::Value& doc) {
  StagedPlan p;
  p.world_size = (int)doc.at("world_size").as_int();
  p.element_size = (int)doc.at("element_size").as_int();
  p.stripe = (int)doc.at("stripe").as_int();
  p.ring = (int)doc.at("ring").as_int();
  p.num_stages = (int)doc.at("num_stages").as_int();
  p.source_program_id = doc.str_or("source_program_id", "");
  for (const auto& b : doc.at("buffers").arr)
    p.buffers[b.at("id").as_str()] = BufferDecl{b.at("length").as_int(), b.bool_or("input", false),
                                                b.bool_or("internal", false)};
  for (const auto& f : doc.at("fences").arr)
    p.fences.push_back(FenceBoundary{(int)f.at("stage").as_int(), f.at("aligned").as_bool()});
  for (const auto& t : doc.at("transfers").arr) p.transfers.push_back(transfer_from_json(t));
  return p;
}

std::string StagedPlan::serialize() const { return json::dump(staged_plan_json(*this)) + "\n"; }

StagedPlan StagedPlan::deserialize(const std::string& text) {
  return staged_plan_from(parse_as(text, "hiercoll-plan-v1"));
}

std::string PipelinedPlan::serialize() const {
  json::Value doc = staged_plan_json(base);
  doc.set("format", json::Value::Str("hiercoll-pipelined-v1"));
  doc.set("pipeline", json::Value::Int(depth));
  doc.set("slots", json::Value::Int(slots));
  return json::dump(doc) + "\n";
}

PipelinedPlan PipelinedPlan::deserialize(const std::string& text) {
  const json::Value doc = parse_as(text, "hiercoll-pipelined-v1");
  PipelinedPlan out;
  out.base = staged_plan_from(doc);
  out.depth = (int)doc.at("pipeline").as_int();
  out.slots = (int)doc.at("slots").as_int();
  return out;
}

}  // namespace hiccl
