// B200 cost model and tuner (see include/hiccl/model.hpp).
#include "hiccl/model.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>

namespace hiccl {

Prediction predict(const PipelinedPlan& plan, int element_size, const B200Model& model,
                   int ranks_per_gpu, int copy_mode) {
  const bool push_copies = copy_mode != 0;
  const bool staged = copy_mode == 2;
  const bool ll = copy_mode == 3;  // tagged lines: 2x the bytes, all pushed
  const int p = plan.base.world_size;
  const int rpg = std::max(1, ranks_per_gpu);
  const int gpus = (p + rpg - 1) / rpg;
  Prediction out;
  out.slot_seconds.assign(std::max(plan.slots, 0), 0.0);
  std::vector<std::vector<const P2PTransfer*>> by_slot(plan.slots);
  for (const auto& t : plan.base.transfers)
    if (t.slot >= 0 && t.slot < plan.slots) by_slot[t.slot].push_back(&t);

  for (int s = 0; s < plan.slots; ++s) {
    if (by_slot[s].empty()) continue;
    // A destination range some transfer reduces into is a pull-reduce
    // group on the device: every remote source of it is loaded by the
    // destination (schedule.cpp); other copies are pushed or pulled.
    std::map<std::tuple<int, std::string, int64_t, int64_t>, bool> reduced;
    for (const P2PTransfer* t : by_slot[s])
      if (t->reduce) reduced[{t->dst, t->dst_buffer, t->dst_offset, t->count}] = true;
    std::vector<double> out_push(gpus, 0), out_pull(gpus, 0), in_push(gpus, 0), in_pull(gpus, 0),
        out_ll(gpus, 0), in_ll(gpus, 0), hbm(gpus, 0);
    for (const P2PTransfer* t : by_slot[s]) {
      double bytes = (double)t->count * element_size;
      const int gs = t->src / rpg, gd = t->dst / rpg;
      if (gs == gd) {
        hbm[gd] += 2 * bytes;
        continue;
      }
      if (ll) {
        out_ll[gs] += 2 * bytes;
        in_ll[gd] += 2 * bytes;
        hbm[gd] += 4 * bytes;  // lines landed, read back, payload stored
        continue;
      }
      const bool in_reduction = reduced.count({t->dst, t->dst_buffer, t->dst_offset, t->count}) > 0;
      const bool pull = (in_reduction && !staged) || !push_copies;
      if (in_reduction && staged) hbm[gd] += 2 * bytes;  // staging write + fold read
      if (pull) {
        in_pull[gd] += bytes;
        out_pull[gs] += bytes;
      } else {
        in_push[gd] += bytes;
        out_push[gs] += bytes;
      }
      hbm[gd] += bytes;  // the landing write
    }
    double busiest = 0;
    for (int g = 0; g < gpus; ++g) {
      const double egress =
          out_push[g] / model.push_bw + out_pull[g] / model.pull_bw + out_ll[g] / model.ll_bw;
      const double ingress =
          in_push[g] / model.push_bw + in_pull[g] / model.pull_bw + in_ll[g] / model.ll_in_bw;
      const double both = (out_ll[g] + in_ll[g]) / model.ll_bidir_bw;
      busiest = std::max({busiest, egress, ingress, both, hbm[g] / model.hbm_bw});
    }
    out.slot_seconds[s] = (ll ? model.ll_step : model.step) + busiest;
    out.seconds += out.slot_seconds[s];
  }
  out.seconds += ll ? model.ll_launch : model.launch;
  return out;
}

TuneChoice tune(CollectiveKind kind, int p, int64_t count, int element_size,
                const B200Model& model) {
  std::vector<Formulation> forms{Formulation::single};
  if (kind == CollectiveKind::broadcast || kind == CollectiveKind::reduce ||
      kind == CollectiveKind::all_gather || kind == CollectiveKind::reduce_scatter ||
      kind == CollectiveKind::all_reduce)
    forms.push_back(Formulation::multi);
  if (kind == CollectiveKind::all_reduce) forms.push_back(Formulation::multi_alt);
  TuneChoice best;
  best.seconds = INFINITY;
  for (Formulation f : forms) {
    CollectiveSpec spec;
    spec.kind = kind;
    spec.formulation = f;
    spec.count = count;
    const CollectiveProgram prog = build(spec, p);
    for (int ring : {1, p}) {
      if (ring > 1 && p < 3) continue;
      MachineDescriptor m = MachineDescriptor::uniform({p}, ring > 1 ? 1 : p);
      for (int depth : {1, 2, 4, 8, 16, 32, 64}) {
        if (count < depth) break;
        try {
          const StagedPlan staged = lower(prog, m, OptimizationConfig{1, ring, depth});
          const PipelinedPlan pp = pipeline(staged, depth);
          for (int mode : {1, 3}) {
            if (mode == 3 && (double)count * element_size * p > 64.0 * (1 << 20)) continue;
            const double t = predict(pp, element_size, model, 1, mode).seconds;
            if (t < best.seconds) best = TuneChoice{f, ring, depth, t, mode};
          }
        } catch (const Error&) {
          // configuration not lowerable (e.g. ring blocks that drop members)
        }
      }
    }
  }
  return best;
}

double t_ring(double alpha, double d, int k, double f, int m, int n, double intra) {
  return (alpha + d / (k * f * m)) * (n + m - 2) + intra / m;
}

double t_tree(double alpha, double d, int k, double f, int m, int n, double intra) {
  int levels = 0;
  while ((1 << levels) < n) ++levels;  // ceil(log2 n)
  return (alpha * m + d / (k * f)) * levels + intra / m;
}

double bound(CollectiveKind kind, int p, int g, int k, double f) {
  if (p <= g)
    throw Error(ErrorCode::NoInterNodeBound,
                "p=" + std::to_string(p) + " fits in one node of g=" + std::to_string(g));
  const double kf = (double)k * f;
  switch (kind) {
    case CollectiveKind::broadcast:
    case CollectiveKind::reduce: return kf;
    case CollectiveKind::gather:
    case CollectiveKind::scatter:
    case CollectiveKind::all_gather:
    case CollectiveKind::reduce_scatter: return kf * p / (p - g);
    case CollectiveKind::all_reduce: return kf * p / (2.0 * (p - g));
    case CollectiveKind::all_to_all: return kf * p / ((double)g * (p - g));
  }
  throw Error(ErrorCode::InvalidConfig, "unknown collective kind");
}

double throughput(double d_bytes, int p, double t) {
  if (t <= 0) throw Error(ErrorCode::InvalidConfig, "t must be positive");
  return d_bytes * p / t;
}

}  // namespace hiccl
