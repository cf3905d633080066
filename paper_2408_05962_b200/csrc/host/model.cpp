// B200 cost model and tuner (see include/hiccl/model.hpp).
#include "hiccl/model.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>

#include "hiccl.h"
#include "layout.hpp"
#include "schedule.hpp"

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
      // a direction whose opposite is idle in this slot runs at the
      // one-direction rates
      const bool in_idle = in_push[g] + in_pull[g] + in_ll[g] == 0;
      const bool out_idle = out_push[g] + out_pull[g] + out_ll[g] == 0;
      const double egress = out_push[g] / (in_idle ? model.push_uni_bw : model.push_bw) +
                            out_pull[g] / (in_idle ? model.pull_uni_bw : model.pull_bw) +
                            out_ll[g] / model.ll_bw;
      const double ingress = in_push[g] / (out_idle ? model.push_uni_bw : model.push_bw) +
                             in_pull[g] / (out_idle ? model.pull_uni_bw : model.pull_bw) +
                             in_ll[g] / model.ll_in_bw;
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

Prediction predict_nvls(const PipelinedPlan& plan, int dtype, const B200Model& model) {
  const int p = plan.base.world_size;
  int esz = 4;
  switch (dtype) {
    case HC_BF16: case HC_F16: esz = 2; break;
    case HC_I64: case HC_F64: esz = 8; break;
    case HC_U8: esz = 1; break;
    default: esz = 4;
  }
  std::vector<int> r2e(p);
  for (int r = 0; r < p; ++r) r2e[r] = r;
  const Schedule s = build_schedule(plan, r2e, p, esz, CopyMode::push);
  LayoutParams lp;
  lp.threads = 256;
  lp.esize = esz;
  lp.ctas = auto_ctas(s, esz, lp.threads, 148);
  lp.dtype = dtype;
  lp.multicast.assign(s.buffer_names.size(), false);
  for (size_t b = 0; b < s.buffer_names.size(); ++b)
    lp.multicast[b] = !s.buffer_decls[b].internal;  // user buffers sit in the window
  std::vector<ExecLayout> layouts;
  for (int e = 0; e < p; ++e) layouts.push_back(build_layout(s, e, lp));
  fuse_nvls(s, layouts);
  Prediction out;
  const int nsteps = layouts.empty() ? 0 : (int)layouts[0].steps.size();
  out.slot_seconds.assign(nsteps, 0.0);
  for (int st = 0; st < nsteps; ++st) {
    std::vector<double> eg_p(p, 0), in_p(p, 0), eg_n(p, 0), in_n(p, 0), res(p, 0), hbm(p, 0);
    bool any = false;
    for (int e = 0; e < p; ++e)
      for (const AbsItem& it : layouts[e].steps[st].items) {
        any = true;
        const double b = (double)it.count * esz;
        const bool red = it.kind == ItemKind::mc_reduce || it.kind == ItemKind::mc_reduce_store;
        const bool mst = it.kind == ItemKind::mc_store || it.kind == ItemKind::mc_reduce_store;
        if (red) {  // the switch reads the range on every member
          for (int g = 0; g < p; ++g) eg_n[g] += b;
          in_n[e] += b;
          res[e] += b;
        }
        if (mst) {  // one copy out, the switch writes every member
          eg_n[e] += b;
          for (int g = 0; g < p; ++g) in_n[g] += b;
        }
        if (it.kind == ItemKind::mc_reduce) {
          const int hd = s.home[it.dst.rank][it.dst.buffer];
          if (hd != e) {  // forwarded straight to another GPU (fuse_forward_copy)
            eg_p[e] += b;
            in_p[hd] += b;
          }
          hbm[hd] += b;
        }
        if (it.kind == ItemKind::mc_store) hbm[e] += b;
        if (it.kind != ItemKind::p2p) continue;
        const int gd = it.dst.rank;
        hbm[gd] += b;
        for (const AbsRef& r : it.srcs) {
          if (r.rank == gd) {
            hbm[gd] += b;
          } else {
            eg_p[r.rank] += b;
            in_p[gd] += b;
          }
        }
      }
    if (!any) continue;
    double busiest = 0;
    for (int g = 0; g < p; ++g) {
      const double eg = eg_p[g] / model.push_bw + eg_n[g] / model.nvls_read_bw;
      const double in = in_p[g] / model.push_bw + in_n[g] / model.nvls_store_bw;
      const double both = (eg_n[g] + in_n[g]) / model.nvls_bidir_bw +
                          (eg_p[g] + in_p[g]) / (2 * model.push_bw);
      busiest = std::max({busiest, eg, in, both, res[g] / model.nvls_reduce_bw, hbm[g] / model.hbm_bw});
    }
    out.slot_seconds[st] = model.step + busiest;
    out.seconds += out.slot_seconds[st];
  }
  out.seconds += model.launch + model.nvls_launch;
  return out;
}

TuneChoice tune_nvls(CollectiveKind kind, int p, int64_t count, int dtype, const B200Model& model) {
  int esz = (dtype == HC_BF16 || dtype == HC_F16) ? 2 : (dtype == HC_I64 || dtype == HC_F64) ? 8
            : dtype == HC_U8 ? 1 : 4;
  TuneChoice best = tune(kind, p, count, esz, model);
  if (p < 2) return best;
  std::vector<Formulation> forms{Formulation::single};
  if (kind == CollectiveKind::broadcast || kind == CollectiveKind::reduce ||
      kind == CollectiveKind::all_gather || kind == CollectiveKind::reduce_scatter ||
      kind == CollectiveKind::all_reduce)
    forms.push_back(Formulation::multi);
  for (Formulation f : forms) {
    CollectiveSpec spec;
    spec.kind = kind;
    spec.formulation = f;
    spec.count = count;
    const CollectiveProgram prog = build(spec, p);
    const MachineDescriptor m = MachineDescriptor::uniform({p}, p);
    for (int depth : {1, 2, 4}) {
      if (count < depth) break;
      try {
        const PipelinedPlan pp = pipeline(lower(prog, m, OptimizationConfig{1, 1, depth}), depth);
        const double t = predict_nvls(pp, dtype, model).seconds;
        if (t < best.seconds) best = TuneChoice{f, 1, depth, t, 1, true};
      } catch (const Error&) {
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
