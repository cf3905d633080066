// Cost model of a pipelined plan on the B200 executor, and a tuner that
// uses it to pick the composition / ring / pipeline depth per message size
// (the paper leaves those knobs to the user).
//
// Same shape as the reference's slot-synchronous simulator
// (proj/src/perf.cpp:48-106): every slot lasts as long as its busiest
// resource plus a latency term. The resources are the B200's: each GPU's
// NVSwitch egress and ingress (point-to-point stores = push, loads = pull
// have different measured ceilings), and its HBM for local traffic. The
// defaults are calibrated on this pool (profiles/r1, tools/nvlinkbench*).
// The reference's closed forms are kept for its acceptance checks:
// Eq. (1) t_ring, Eq. (2) t_tree, Table 4 bounds, d*p/t throughput
// (perf.cpp:108-140).
#pragma once

#include <string>
#include <vector>

#include "hiccl/plan.hpp"
#include "hiccl/presets.hpp"

namespace hiccl {

struct B200Model {
  double launch = 10.5e-6;     // kernel launch + entry/exit barriers (s)
  double step = 3.5e-6;        // flag round per dependent step (s)
  double push_bw = 691e9;      // all-to-all peer stores, per GPU per direction (B/s)
  double pull_bw = 650e9;      // all-to-all peer loads, per GPU per direction
  // one direction of a GPU's links busy, the other idle (tools/nvlinkbench.cu:
  // peer read 775, peer write 712 GB/s)
  double pull_uni_bw = 770e9;
  double push_uni_bw = 710e9;
  double hbm_bw = 5.8e12;      // executor's local copy rate, read+write bytes/s
  double ll_launch = 4e-6;     // tagged-line mode: launch, no barriers
  double ll_step = 3e-6;       // tagged-line mode: one store-to-poll exchange
  double ll_bw = 530e9;        // tagged-line mode: line bytes (2x payload) a GPU stores to peers
  double ll_in_bw = 700e9;     // tagged-line mode: line bytes a GPU receives
  double ll_bidir_bw = 600e9;  // tagged-line mode: line bytes stored + received (both ways busy)
  // NVLS library (multimem, tools/nvlsbench.cu, profiles/r1/nvls): bytes a
  // GPU serves to switch reads (ld_reduce), bytes multicast stores land on
  // it, and the sum of both when both directions are busy (fused all-reduce)
  double nvls_read_bw = 705e9;
  double nvls_store_bw = 715e9;
  double nvls_bidir_bw = 1158e9;
  double nvls_reduce_bw = 455e9;  // ld_reduce results one GPU draws (single-issuer reduce)
  // extra fixed cost of a launch with multimem items: the proxy fences
  // after every acquire (broadcast 1 MiB 19.4 us against 15.3 without them,
  // profiles/r2/alias_fence_cost.txt)
  double nvls_launch = 4.5e-6;
};

struct Prediction {
  double seconds = 0;
  std::vector<double> slot_seconds;
};

/// Predicted time of one start()/wait() of `plan` with `ranks_per_gpu`
/// logical ranks on every GPU (contiguous); copy_mode 0 pull, 1 push,
/// 2 staged, 3 ll (as hc_exec_config::copy_mode).
Prediction predict(const PipelinedPlan& plan, int element_size, const B200Model& model,
                   int ranks_per_gpu = 1, int copy_mode = 1);

/// Predicted time with the user buffers in an NVLS window (one rank per
/// GPU): the executors' own device layout (multimem lowering and the
/// reduce+multicast fusion, layout.hpp) costed per device step; dtype is an
/// hc_dtype code (it decides which reductions the switch can do).
Prediction predict_nvls(const PipelinedPlan& plan, int dtype, const B200Model& model);

struct TuneChoice {
  Formulation formulation = Formulation::single;
  int ring = 1;       // with g = 1 when > 1 (one "node" per GPU)
  int pipeline = 1;
  double seconds = 0;
  int copy_mode = 1;  // 1 push or 3 ll (hc_exec_config::copy_mode)
  bool nvls = false;  // buffers in an NVLS window (library "NVLS")
};

/// Best (formulation, ring, pipeline, copy mode) for a preset collective of
/// `count` elements per rank chunk on flat {p}, by the model. Tagged lines
/// are considered while the per-rank buffer is at most 64 MiB (their
/// staging is 4x the landed bytes).
TuneChoice tune(CollectiveKind kind, int p, int64_t count, int element_size,
                const B200Model& model = B200Model());

/// Same, also considering the NVLS library (flat {p}, ring 1) for dtype.
TuneChoice tune_nvls(CollectiveKind kind, int p, int64_t count, int dtype,
                     const B200Model& model = B200Model());

// ---- the reference's analytic forms (perf.cpp:108-140) ----
double t_ring(double alpha, double d, int k, double f, int m, int n, double intra);
double t_tree(double alpha, double d, int k, double f, int m, int n, double intra);
double bound(CollectiveKind kind, int p, int g, int k, double f);  // NoInterNodeBound if p <= g
double throughput(double d_bytes, int p, double t);

}  // namespace hiccl
