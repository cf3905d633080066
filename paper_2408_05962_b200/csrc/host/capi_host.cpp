// C ABI: composition and lowering entry points (include/hiccl.h).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "capi_common.hpp"
#include "json.hpp"
#include "layout.hpp"
#include "schedule.hpp"
#include "hiccl/plan.hpp"
#include "hiccl/model.hpp"
#include "hiccl/presets.hpp"

struct hc_program {
  hiccl::CollectiveProgram prog;
};

struct hc_plan {
  hiccl::PipelinedPlan plan;
  std::vector<std::string> buffer_names;  // map order
  std::vector<hiccl::BufferDecl> buffer_decls;
  void index() {
    buffer_names.clear();
    buffer_decls.clear();
    for (const auto& [name, d] : plan.base.buffers) {
      buffer_names.push_back(name);
      buffer_decls.push_back(d);
    }
  }
};

namespace hiccl::capi {

thread_local std::string g_last_error;

char* dup_string(const std::string& s) {
  char* p = (char*)std::malloc(s.size() + 1);
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

MachineDescriptor machine_from(const hc_machine_desc* d) {
  if (!d || !d->hierarchy || d->num_levels < 1)
    throw Error(ErrorCode::InvalidMachine, "machine description missing");
  std::vector<int> h(d->hierarchy, d->hierarchy + d->num_levels);
  MachineDescriptor m = MachineDescriptor::uniform(h, d->gpus_per_node);
  if (d->transport)
    for (int i = 0; i < d->num_levels; ++i)
      if (d->transport[i]) m.set_transport(i, d->transport[i]);
  return m;
}

const PipelinedPlan& plan_of(const hc_plan* p) { return p->plan; }

}  // namespace hiccl::capi

using namespace hiccl;
using hiccl::capi::guard;

extern "C" {

const char* hc_last_error(void) { return capi::g_last_error.c_str(); }
void hc_free(void* p) { std::free(p); }
const char* hc_version(void) { return "hiccl-b200 0.1"; }

hc_status hc_program_create(int world_size, hc_program** out) {
  return guard([&] { *out = new hc_program{CollectiveProgram(world_size)}; });
}

void hc_program_destroy(hc_program* prog) { delete prog; }

hc_status hc_program_declare_buffer(hc_program* prog, const char* id, int64_t length,
                                    int input, int internal) {
  return guard([&] { prog->prog.declare_buffer(id, length, input != 0, internal != 0); });
}

hc_status hc_program_add_multicast(hc_program* prog, const char* send_buf, int64_t send_off,
                                   const char* recv_buf, int64_t recv_off, int64_t count,
                                   int root, const int* leaves, int n_leaves) {
  return guard([&] {
    prog->prog.add_multicast(BufferRef{send_buf, send_off, count},
                             BufferRef{recv_buf, recv_off, count}, root,
                             std::vector<Rank>(leaves, leaves + std::max(0, n_leaves)));
  });
}

hc_status hc_program_add_reduction(hc_program* prog, const char* send_buf, int64_t send_off,
                                   const char* recv_buf, int64_t recv_off, int64_t count,
                                   const int* leaves, int n_leaves, int root, int op) {
  return guard([&] {
    if (op != HC_OP_SUM && op != HC_OP_MAX) throw Error(ErrorCode::ParseError, "unknown op");
    prog->prog.add_reduction(BufferRef{send_buf, send_off, count},
                             BufferRef{recv_buf, recv_off, count},
                             std::vector<Rank>(leaves, leaves + std::max(0, n_leaves)), root,
                             (ReduceOp)op);
  });
}

hc_status hc_program_add_fence(hc_program* prog) {
  return guard([&] { prog->prog.add_fence(); });
}

hc_status hc_program_validate(const hc_program* prog, char** report) {
  return guard([&] {
    std::string s;
    for (const auto& v : prog->prog.validate())
      s += to_string(v.code) + "|" + std::to_string(v.step) + "|" + std::to_string(v.primitive) +
           "|" + std::to_string(v.rank) + "|" + v.buffer + "|" + std::to_string(v.lo) + "|" +
           std::to_string(v.hi) + "|" + v.message + "\n";
    *report = capi::dup_string(s);
  });
}

hc_status hc_program_serialize(const hc_program* prog, char** json) {
  return guard([&] { *json = capi::dup_string(prog->prog.serialize()); });
}

hc_status hc_program_deserialize(const char* json, hc_program** out) {
  return guard([&] { *out = new hc_program{CollectiveProgram::deserialize(json)}; });
}

hc_status hc_program_id(const hc_program* prog, char** id) {
  return guard([&] { *id = capi::dup_string(prog->prog.id()); });
}

hc_status hc_program_preset(int kind, int formulation, int p, int64_t count, int root, int op,
                            hc_program** out) {
  return guard([&] {
    if (kind < 0 || kind > 7) throw Error(ErrorCode::ParseError, "unknown collective kind");
    if (formulation < 0 || formulation > 2) throw Error(ErrorCode::ParseError, "unknown formulation");
    CollectiveSpec spec;
    spec.kind = (CollectiveKind)kind;
    spec.formulation = (Formulation)formulation;
    spec.count = count;
    spec.root = root;
    spec.op = (ReduceOp)op;
    *out = new hc_program{build(spec, p)};
  });
}

hc_status hc_plan_lower(const hc_program* prog, const hc_machine_desc* machine, int ring,
                        int stripe, int pipeline_depth, hc_plan** out) {
  return guard([&] {
    auto m = capi::machine_from(machine);
    auto staged = lower(prog->prog, m, OptimizationConfig{stripe, ring, pipeline_depth});
    auto* p = new hc_plan{pipeline(staged, pipeline_depth), {}, {}};
    p->index();
    *out = p;
  });
}

hc_status hc_plan_lower_staged_json(const hc_program* prog, const hc_machine_desc* machine,
                                    int ring, int stripe, char** json) {
  return guard([&] {
    auto m = capi::machine_from(machine);
    *json = capi::dup_string(lower(prog->prog, m, OptimizationConfig{stripe, ring, 1}).serialize());
  });
}

hc_status hc_plan_serialize(const hc_plan* plan, char** json) {
  return guard([&] { *json = capi::dup_string(plan->plan.serialize()); });
}

hc_status hc_plan_deserialize(const char* json, hc_plan** out) {
  return guard([&] {
    auto* p = new hc_plan{PipelinedPlan::deserialize(json), {}, {}};
    p->index();
    *out = p;
  });
}

void hc_plan_destroy(hc_plan* plan) { delete plan; }

hc_status hc_plan_get_info(const hc_plan* plan, hc_plan_info* out) {
  return guard([&] {
    const auto& pp = plan->plan;
    out->world_size = pp.base.world_size;
    out->num_transfers = (int)pp.base.transfers.size();
    out->num_buffers = (int)plan->buffer_names.size();
    out->num_stages = pp.base.num_stages;
    out->slots = pp.slots;
    out->depth = pp.depth;
    out->stripe = pp.base.stripe;
    out->ring = pp.base.ring;
  });
}

hc_status hc_plan_get_buffer(const hc_plan* plan, int index, const char** name, int64_t* length,
                             int* input, int* internal) {
  return guard([&] {
    if (index < 0 || index >= (int)plan->buffer_names.size())
      throw Error(ErrorCode::BadBufferRef, "buffer index out of range");
    *name = plan->buffer_names[index].c_str();
    *length = plan->buffer_decls[index].length;
    *input = plan->buffer_decls[index].input;
    *internal = plan->buffer_decls[index].internal;
  });
}

hc_status hc_plan_get_transfers(const hc_plan* plan, hc_transfer* out) {
  return guard([&] {
    std::map<std::string, int> ids;
    for (size_t i = 0; i < plan->buffer_names.size(); ++i) ids[plan->buffer_names[i]] = (int)i;
    for (const auto& t : plan->plan.base.transfers) {
      hc_transfer& r = out[t.id];
      r.id = t.id;
      r.src = t.src;
      r.dst = t.dst;
      r.src_buf = ids.at(t.src_buffer);
      r.dst_buf = ids.at(t.dst_buffer);
      r.reduce = t.reduce;
      r.op = (int)t.op;
      r.stage = t.stage;
      r.slot = t.slot;
      r.channel = t.channel;
      r.stripe = t.stripe;
      r.level = t.level;
      r.step = t.step;
      r.n_deps = (int)t.deps.size();
      r.src_off = t.src_offset;
      r.dst_off = t.dst_offset;
      r.count = t.count;
    }
  });
}

hc_status hc_plan_comm_matrix(const hc_plan* plan, int slot, int64_t* out) {
  return guard([&] {
    auto m = comm_matrix(plan->plan, slot);
    const size_t p = m.size();
    for (size_t i = 0; i < p; ++i)
      for (size_t j = 0; j < p; ++j) out[i * p + j] = m[i][j];
  });
}

hc_status hc_plan_layout_summary(const hc_plan* plan, int num_execs, const int* rank_to_exec,
                                 int copy_mode, int dtype, int ctas, const char* multicast_buffers,
                                 char** out) {
  return guard([&] {
    const int p = plan->plan.base.world_size;
    std::vector<int> r2e = rank_to_exec ? std::vector<int>(rank_to_exec, rank_to_exec + p)
                                        : std::vector<int>(p, 0);
    int esize = 0;
    switch (dtype) {
      case HC_F32: case HC_I32: esize = 4; break;
      case HC_BF16: case HC_F16: esize = 2; break;
      case HC_I64: case HC_F64: esize = 8; break;
      case HC_U8: esize = 1; break;
      default: throw Error(ErrorCode::InvalidConfig, "unknown dtype");
    }
    Schedule s = build_schedule(plan->plan, r2e, num_execs, esize,
                                (CopyMode)std::max(0, std::min(3, copy_mode)));
    LayoutParams lp;
    lp.threads = s.ll ? 256 : 512;
    lp.esize = esize;
    lp.ctas = ctas > 0 ? ctas : auto_ctas(s, esize, lp.threads, 148);
    lp.dtype = dtype;
    lp.alt_halves = want_alt_halves(s, esize);
    if (const char* ah = std::getenv("HICCL_ALT_HALVES")) lp.alt_halves = atoi(ah) != 0;
    lp.multicast.assign(s.buffer_names.size(), false);
    if (const char* ts = std::getenv("HICCL_TILE_SYNC")) lp.tile_sync = atoi(ts) != 0;
    std::string names = multicast_buffers ? multicast_buffers : "";
    for (size_t a = 0; a < names.size();) {
      size_t b = names.find(',', a);
      if (b == std::string::npos) b = names.size();
      const std::string n = names.substr(a, b - a);
      for (size_t k = 0; k < s.buffer_names.size(); ++k)
        if (s.buffer_names[k] == n) lp.multicast[k] = true;
      a = b + 1;
    }
    std::vector<ExecLayout> layouts;
    for (int e = 0; e < num_execs; ++e) layouts.push_back(build_layout(s, e, lp));
    const int fused = fuse_nvls(s, layouts);
    const auto sync = analyze_sync(s, layouts, lp);
    verify_sync(s, layouts, sync, lp);
    static const char* kinds[] = {"p2p", "mc_reduce", "mc_store", "mc_reduce_store"};
    json::Value j = json::Value::Obj();
    j.set("fused", json::Value::Int(fused));
    j.set("alt_halves", json::Value::Bool(lp.alt_halves));
    j.set("ctas", json::Value::Int(lp.ctas));
    json::Value ex = json::Value::Arr();
    for (int e = 0; e < num_execs; ++e) {
      json::Value steps = json::Value::Arr();
      for (const StepLayout& L : layouts[e].steps) {
        json::Value st = json::Value::Arr();
        for (const AbsItem& it : L.items) st.push(json::Value::Str(kinds[(int)it.kind]));
        steps.push(std::move(st));
      }
      // tiles per CTA: the busiest CTA of each step bounds the step
      json::Value peak = json::Value::Arr();
      for (const StepLayout& L : layouts[e].steps) {
        std::vector<int64_t> n(L.cta_n, 0);
        for (const AbsItem& it : L.items)
          for (uint32_t l = 0; l < it.n_tiles; ++l) ++n[(it.base_cta + l) % (uint32_t)L.cta_n];
        peak.push(json::Value::Int(n.empty() ? 0 : *std::max_element(n.begin(), n.end())));
      }
      json::Value tiles = json::Value::Arr();
      for (const StepLayout& L : layouts[e].steps) tiles.push(json::Value::Int(L.n_tiles));
      json::Value o = json::Value::Obj();
      o.set("steps", std::move(steps));
      o.set("cta_peak_tiles", std::move(peak));
      o.set("tiles", std::move(tiles));
      o.set("paired_waits", json::Value::Int(sync[e].paired));
      o.set("whole_waits", json::Value::Int(sync[e].whole));
      ex.push(std::move(o));
    }
    j.set("execs", std::move(ex));
    *out = capi::dup_string(json::dump(j));
  });
}

namespace {
void corrupt_schedule(Schedule& s, int mode) {
  for (auto& w : s.items) {
    const size_t first = w.reads_dst ? 1 : 0;  // a live destination stays first
    if (mode == 1 && w.srcs.size() >= first + 2) {
      std::swap(w.srcs[w.srcs.size() - 1], w.srcs[w.srcs.size() - 2]);
      return;
    }
    if (mode == 2 && w.srcs.size() >= 2) {
      w.srcs.pop_back();
      return;
    }
    if (mode == 3 && w.count >= 2) {
      for (auto& l : w.srcs) l.offset += 1;
      w.dst.offset += 1;
      w.count -= 1;
      return;
    }
  }
  throw Error(ErrorCode::InvalidConfig, "no item to damage");
}
}  // namespace

hc_status hc_plan_schedule_summary(const hc_plan* plan, int num_execs, const int* rank_to_exec,
                                   int copy_mode, int element_size, int verify, char** out) {
  return guard([&] {
    const int p = plan->plan.base.world_size;
    std::vector<int> r2e = rank_to_exec ? std::vector<int>(rank_to_exec, rank_to_exec + p)
                                        : std::vector<int>(p, 0);
    Schedule s = build_schedule(plan->plan, r2e, num_execs, element_size,
                                (CopyMode)std::max(0, std::min(3, copy_mode)));
    // verify: 1 full check, 2 the segment replay alone; 16 + m first
    // damages the schedule (negative tests of the checker): m = 1 swaps the
    // last two sources of a fold, 2 drops the last source, 3 shortens an
    // item by its first element
    if (verify >= 16) corrupt_schedule(s, verify - 16);
    if (verify == 2) {
      if (!replay_schedule(plan->plan, s, 1LL << 26))
        throw Error(ErrorCode::InvalidConfig, "schedule too fragmented to replay");
    } else if (verify) {
      verify_schedule(plan->plan, s);
    }
    // device layout + tile-granular sync as the executors would build it
    // (G = 148 CTAs or fewer for small plans, 512 threads, no NVLS)
    LayoutParams lp;
    lp.threads = s.ll ? 256 : 512;
    lp.esize = element_size;
    lp.ctas = auto_ctas(s, element_size, lp.threads, 148);
    lp.dtype = 0;
    lp.multicast.assign(s.buffer_names.size(), false);
    if (const char* ts = std::getenv("HICCL_TILE_SYNC")) lp.tile_sync = atoi(ts) != 0;
    std::vector<ExecLayout> layouts;
    for (int e = 0; e < num_execs; ++e) layouts.push_back(build_layout(s, e, lp));
    const auto sync = analyze_sync(s, layouts, lp);
    if (verify && verify != 2) verify_sync(s, layouts, sync, lp);
    json::Value j = json::Value::Obj();
    j.set("steps", json::Value::Int((int64_t)s.step_slot.size()));
    j.set("items", json::Value::Int((int64_t)s.items.size()));
    j.set("max_sources", json::Value::Int(s.max_sources));
    j.set("max_phases", json::Value::Int(s.max_phases));
    j.set("ctas", json::Value::Int(lp.ctas));
    json::Value ex = json::Value::Arr();
    for (int e = 0; e < num_execs; ++e) {
      const auto& ep = s.execs[e];
      int64_t n_items = 0, n_waits = 0, n_pub = 0, remote_waits = 0;
      for (size_t k = 0; k < ep.items_by_step.size(); ++k) {
        n_items += (int64_t)ep.items_by_step[k].size();
        n_waits += (int64_t)ep.waits[k].size();
        for (const auto& w : ep.waits[k]) remote_waits += w.exec != e;
        n_pub += ep.publish[k];
      }
      json::Value o = json::Value::Obj();
      o.set("items", json::Value::Int(n_items));
      o.set("waits", json::Value::Int(n_waits));
      o.set("remote_waits", json::Value::Int(remote_waits));
      o.set("publish", json::Value::Int(n_pub));
      o.set("arena_bytes", json::Value::Int(s.arena_bytes[e]));
      o.set("paired_waits", json::Value::Int(sync[e].paired));
      o.set("whole_waits", json::Value::Int(sync[e].whole));
      int64_t sys_pub = 0;
      for (uint8_t v : sync[e].publish) sys_pub += v == 2;
      o.set("sys_publish", json::Value::Int(sys_pub));
      ex.push(std::move(o));
    }
    j.set("execs", std::move(ex));
    json::Value items = json::Value::Arr();
    for (const auto& w : s.items) {
      json::Value o = json::Value::Obj();
      o.set("step", json::Value::Int(w.step));
      o.set("exec", json::Value::Int(w.exec));
      o.set("dst_rank", json::Value::Int(w.dst.rank));
      o.set("dst_buffer", json::Value::Str(s.buffer_names[w.dst.buffer]));
      o.set("dst_offset", json::Value::Int(w.dst.offset));
      o.set("dst_home", json::Value::Int(s.home[w.dst.rank][w.dst.buffer]));
      o.set("count", json::Value::Int(w.count));
      o.set("reads_dst", json::Value::Bool(w.reads_dst));
      o.set("n_src", json::Value::Int((int64_t)w.srcs.size()));
      o.set("transfers", json::Value::IntArr(w.transfer_ids));
      items.push(std::move(o));
    }
    j.set("item_list", std::move(items));
    *out = capi::dup_string(json::dump(j));
  });
}

static B200Model model_from(const hc_model* m) {
  B200Model b;
  if (m) {
    b.launch = m->launch;
    b.step = m->step;
    b.push_bw = m->push_bw;
    b.pull_bw = m->pull_bw;
    b.hbm_bw = m->hbm_bw;
    b.ll_launch = m->ll_launch;
    b.ll_step = m->ll_step;
    b.ll_bw = m->ll_bw;
    b.ll_in_bw = m->ll_in_bw;
    b.ll_bidir_bw = m->ll_bidir_bw;
    b.nvls_read_bw = m->nvls_read_bw;
    b.nvls_store_bw = m->nvls_store_bw;
    b.nvls_bidir_bw = m->nvls_bidir_bw;
    b.nvls_reduce_bw = m->nvls_reduce_bw;
    b.pull_uni_bw = m->pull_uni_bw;
    b.push_uni_bw = m->push_uni_bw;
    b.nvls_launch = m->nvls_launch;
  }
  return b;
}

hc_status hc_model_default(hc_model* out) {
  return guard([&] {
    B200Model b;
    *out = hc_model{b.launch,   b.step,      b.push_bw,       b.pull_bw,
                    b.hbm_bw,   b.ll_launch, b.ll_step,       b.ll_bw,
                    b.ll_in_bw, b.ll_bidir_bw, b.nvls_read_bw, b.nvls_store_bw,
                    b.nvls_bidir_bw, b.nvls_reduce_bw, b.pull_uni_bw, b.push_uni_bw,
                    b.nvls_launch};
  });
}

hc_status hc_plan_predict(const hc_plan* plan, int element_size, const hc_model* model,
                          int ranks_per_gpu, int copy_mode, double* seconds) {
  return guard([&] {
    *seconds = predict(plan->plan, element_size, model_from(model), ranks_per_gpu,
                       std::max(0, std::min(3, copy_mode))).seconds;
  });
}

hc_status hc_tune(int kind, int p, int64_t count, int element_size, const hc_model* model,
                  hc_tune_result* out) {
  return guard([&] {
    if (kind < 0 || kind > 7) throw Error(ErrorCode::ParseError, "unknown collective kind");
    TuneChoice c = tune((CollectiveKind)kind, p, count, element_size, model_from(model));
    *out = hc_tune_result{(int)c.formulation, c.ring, c.pipeline, c.seconds, c.copy_mode, 0};
  });
}

hc_status hc_plan_predict_nvls(const hc_plan* plan, int dtype, const hc_model* model,
                               double* seconds) {
  return guard([&] { *seconds = predict_nvls(plan->plan, dtype, model_from(model)).seconds; });
}

hc_status hc_tune_nvls(int kind, int p, int64_t count, int dtype, const hc_model* model,
                       hc_tune_result* out) {
  return guard([&] {
    if (kind < 0 || kind > 7) throw Error(ErrorCode::ParseError, "unknown collective kind");
    TuneChoice c = tune_nvls((CollectiveKind)kind, p, count, dtype, model_from(model));
    *out = hc_tune_result{(int)c.formulation, c.ring, c.pipeline, c.seconds, c.copy_mode,
                          c.nvls ? 1 : 0};
  });
}

hc_status hc_t_ring(double alpha, double d, int k, double f, int m, int n, double intra,
                    double* seconds) {
  return guard([&] { *seconds = t_ring(alpha, d, k, f, m, n, intra); });
}

hc_status hc_t_tree(double alpha, double d, int k, double f, int m, int n, double intra,
                    double* seconds) {
  return guard([&] { *seconds = t_tree(alpha, d, k, f, m, n, intra); });
}

hc_status hc_bound(int kind, int p, int g, int k, double f, double* out) {
  return guard([&] {
    if (kind < 0 || kind > 7) throw Error(ErrorCode::ParseError, "unknown collective kind");
    *out = bound((CollectiveKind)kind, p, g, k, f);
  });
}

hc_status hc_throughput(double d_bytes, int p, double t, double* out) {
  return guard([&] { *out = throughput(d_bytes, p, t); });
}

}  // extern "C"
