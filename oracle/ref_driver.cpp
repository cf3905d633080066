// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// A thin C-ABI driver over the *unmodified* reference library
// (`hiercoll`, compiled from /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/). Only tests/, __graft_entry__.smoke() and bench.py's
// reference / cpu_baseline legs may load it, and only as the checker.
//
// What it exposes (all strings are malloc'd; free with ref_free):
//   ref_preset_pipelined_json  build(spec,p) -> lower -> pipeline -> serialize
//                              (presets.cpp:89, factorize.cpp:587,
//                               pipeline.cpp:76, pipeline.cpp:147)
//   ref_program_json           build(spec,p).serialize()  (composition.cpp:363)
//   ref_lower_program_json     deserialize(program) -> lower -> pipeline
//   ref_check_pipelined_json   deserialize(pipelined plan) -> execute_plan ->
//                              states_equal(reference_semantics)
//                              (engine.cpp:341, presets.cpp:231, engine.cpp:221)
//   ref_check_program_plan     execute_plan(plan) vs execute_program(program)
//   ref_time_execute_plan      wall time of the reference executor
//                              (engine.cpp:285-330) for the reference arm
//   ref_simulate_json          perf.cpp:48 simulate() total seconds
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hiercoll/composition.hpp"
#include "hiercoll/engine.hpp"
#include "hiercoll/factorize.hpp"
#include "hiercoll/machine.hpp"
#include "hiercoll/perf.hpp"
#include "hiercoll/pipeline.hpp"
#include "hiercoll/presets.hpp"

using namespace hiercoll;

namespace {

char* dup(const std::string& s) {
  char* p = (char*)std::malloc(s.size() + 1);
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

// Same uniform fixture as tests/test_common.hpp:25-38 of the reference.
MachineDescriptor make_machine(const int* hier, int nlev, int g) {
  MachineDescriptor m;
  m.hierarchy.assign(hier, hier + nlev);
  for (int i = 0; i < nlev; ++i) m.levels.push_back(LevelLink{1e-6, 100e9, "sim"});
  m.gpus_per_node = g;
  m.nics_per_node = 1;
  m.nic_bandwidth = 25e9;
  m.binding = Binding::packed;
  m.element_size = 4;
  return m;
}

CollectiveSpec make_spec(int kind, int form, int64_t count, int root, int op) {
  CollectiveSpec s;
  s.kind = (CollectiveKind)kind;
  s.formulation = (Formulation)form;
  s.count = count;
  s.root = root;
  s.op = (ReduceOp)op;
  return s;
}

// Returns 0 on success; on a hiercoll::Error returns 1 + (int)code and
// stores "Code: message" in *err.
template <class F>
int guarded(char** err, F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    if (err) *err = dup(e.what());
    return 1 + (int)e.code();
  } catch (const std::exception& e) {
    if (err) *err = dup(e.what());
    return 100;
  }
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

int ref_program_json(int kind, int form, int p, int64_t count, int root, int op,
                     char** out, char** err) {
  return guarded(err, [&] { *out = dup(build(make_spec(kind, form, count, root, op), p).serialize()); });
}

int ref_preset_pipelined_json(int kind, int form, int p, int64_t count, int root,
                              int op, const int* hier, int nlev, int g,
                              int stripe, int ring, int depth, char** out,
                              char** err) {
  return guarded(err, [&] {
    auto prog = build(make_spec(kind, form, count, root, op), p);
    auto m = make_machine(hier, nlev, g);
    auto plan = lower(prog, m, OptimizationConfig{stripe, ring, depth});
    *out = dup(pipeline(plan, depth).serialize());
  });
}

int ref_preset_staged_json(int kind, int form, int p, int64_t count, int root,
                           int op, const int* hier, int nlev, int g, int stripe,
                           int ring, char** out, char** err) {
  return guarded(err, [&] {
    auto prog = build(make_spec(kind, form, count, root, op), p);
    auto m = make_machine(hier, nlev, g);
    *out = dup(lower(prog, m, OptimizationConfig{stripe, ring, 1}).serialize());
  });
}

int ref_lower_program_json(const char* program_json, const int* hier, int nlev,
                           int g, int stripe, int ring, int depth, char** out,
                           char** err) {
  return guarded(err, [&] {
    auto prog = CollectiveProgram::deserialize(program_json);
    auto m = make_machine(hier, nlev, g);
    auto plan = lower(prog, m, OptimizationConfig{stripe, ring, depth});
    *out = dup(pipeline(plan, depth).serialize());
  });
}

int ref_roundtrip_program_json(const char* program_json, char** out, char** err) {
  return guarded(err, [&] { *out = dup(CollectiveProgram::deserialize(program_json).serialize()); });
}

// Validate a serialized program; returns violations as "Code|step|prim\n" lines.
int ref_validate_program_json(const char* program_json, char** out, char** err) {
  return guarded(err, [&] {
    auto prog = CollectiveProgram::deserialize(program_json);
    std::string s;
    for (const auto& v : prog.validate())
      s += to_string(v.code) + "|" + std::to_string(v.step) + "|" +
           std::to_string(v.primitive) + "\n";
    *out = dup(s);
  });
}

// 0 = PASS; 1 = divergence (message in *out); >1 = error code + 1.
int ref_check_pipelined_json(const char* plan_json, int kind, int form, int p,
                             int64_t count, int root, int op, char** out,
                             char** err) {
  int diverged = 0;
  int rc = guarded(err, [&] {
    auto pp = PipelinedPlan::deserialize(plan_json);
    auto actual = execute_plan(pp);
    auto expect = reference_semantics(make_spec(kind, form, count, root, op), p);
    auto d = states_equal(expect, actual);
    if (d) {
      diverged = 1;
      *out = dup(d->to_string());
    } else {
      *out = dup("PASS");
    }
  });
  if (rc) return rc + 1;
  return diverged;
}

int ref_check_program_plan(const char* program_json, const char* plan_json,
                           char** out, char** err) {
  int diverged = 0;
  int rc = guarded(err, [&] {
    auto prog = CollectiveProgram::deserialize(program_json);
    auto pp = PipelinedPlan::deserialize(plan_json);
    auto d = states_equal(execute_program(prog), execute_plan(pp));
    diverged = d ? 1 : 0;
    *out = dup(d ? d->to_string() : std::string("PASS"));
  });
  if (rc) return rc + 1;
  return diverged;
}

// Wall seconds of the reference executor alone (execute_plan,
// engine.cpp:334-347) on the pipelined plan of a preset collective.
int ref_time_execute_plan(int kind, int form, int p, int64_t count, int root,
                          int op, const int* hier, int nlev, int g, int stripe,
                          int ring, int depth, double* seconds, char** err) {
  return guarded(err, [&] {
    auto prog = build(make_spec(kind, form, count, root, op), p);
    auto m = make_machine(hier, nlev, g);
    auto pp = pipeline(lower(prog, m, OptimizationConfig{stripe, ring, depth}), depth);
    auto t0 = std::chrono::steady_clock::now();
    auto st = execute_plan(pp);
    auto t1 = std::chrono::steady_clock::now();
    (void)st;
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

int ref_simulate_seconds(const char* plan_json, const int* hier, int nlev, int g,
                         double* seconds, char** err) {
  return guarded(err, [&] {
    auto pp = PipelinedPlan::deserialize(plan_json);
    auto m = make_machine(hier, nlev, g);
    *seconds = simulate(pp, m).total;
  });
}

int ref_inter_node_bytes(const char* staged_json, int node_size, int64_t* bytes,
                         char** err) {
  return guarded(err, [&] {
    *bytes = inter_node_bytes(StagedPlan::deserialize(staged_json), node_size);
  });
}

}  // extern "C"
