#!/usr/bin/env python
"""Render the graph-replayed sweeps (tools/run_graph_evidence.sh) as a
markdown table: per collective and size, NCCL, hiccl's auto choice (cost
model), and each fixed mode.

  python tools/summarize_graph.py profiles/r1/graph > profiles/r1/GRAPH_SUMMARY.md
"""
import glob
import json
import sys
from collections import defaultdict


def size(b):
    for u, n in (("GiB", 1 << 30), ("MiB", 1 << 20), ("KiB", 1 << 10)):
        if b >= n:
            return f"{b // n} {u}"
    return f"{b} B"


def main(d):
    print("# Graph-replayed sweeps (round 1)\n")
    print("50 launches captured in one CUDA graph per rank, replayed once after a warm-up "
          "replay; time = max over ranks of the replay / 50 (CUDA events). NCCL 2.28.9 "
          "through torch.distributed, captured the same way. fp32, flat {p}, one process "
          "per GPU. `auto` = the cost model's formulation and copy mode "
          "(`H.tune`, s = single, m = multi). Times in µs; lower is better.\n")
    for p in (4, 2):
        rows = [json.loads(l) for f in sorted(glob.glob(f"{d}/*_p{p}*.jsonl")) for l in open(f)]
        best = defaultdict(dict)
        for r in rows:
            if "us" not in r:
                continue
            key = (r["collective"], r["bytes"])
            if r["impl"] == "nccl":
                best[key]["nccl"] = r["us"]
            elif r.get("auto"):
                best[key]["auto"] = (r["us"], r["formulation"][0] + "/" + r["copy_mode"])
            else:
                rooted = r["collective"] in ("all_reduce", "broadcast", "reduce")
                tag = r["copy_mode"] + ("/" + r["formulation"][0] if rooted else "")
                best[key][tag] = r["us"]
        print(f"\n## p = {p}\n")
        print("| collective | S | NCCL | hiccl auto | choice | auto / NCCL | fixed modes |")
        print("|---|---|---|---|---|---|---|")
        for key in sorted(best):
            v = best[key]
            nccl = v.get("nccl")
            a, choice = v.get("auto", (None, ""))
            others = ", ".join(f"{k} {x:.1f}" for k, x in sorted(v.items()) if k not in ("nccl", "auto"))
            ratio = f"{a / nccl:.2f}" if a and nccl else "—"
            print(f"| {key[0]} | {size(key[1])} | {nccl and round(nccl, 1) or '—'} | "
                  f"{a and round(a, 1)} | {choice} | {ratio} | {others} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r1/graph")
