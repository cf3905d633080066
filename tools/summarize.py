#!/usr/bin/env python
"""Render profiles/<round>/SUMMARY.md tables from the sweep JSONL files."""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r1")


def fmt_b(b):
    return f"{b >> 30} GiB" if b >= 1 << 30 else f"{b >> 20} MiB" if b >= 1 << 20 else f"{b >> 10} KiB"


def rows(f):
    return [json.loads(l) for l in open(f)] if Path(f).exists() else []


out = []
for p in (2, 4):
    tab = {}
    for r in rows(d / f"sweep_p{p}.jsonl"):
        tab.setdefault((r["collective"], r["bytes"]), {})[r["impl"]] = r
    if not tab:
        continue
    out.append(f"## p = {p}: all eight collectives vs NCCL\n")
    out.append("| collective | S | hiccl µs | hiccl busbw GB/s | NCCL µs | NCCL busbw GB/s | NCCL time / hiccl time |")
    out.append("|---|---|---|---|---|---|---|")
    for (c, b), v in sorted(tab.items()):
        h, n = v.get("hiccl"), v.get("nccl")
        if not h or "us" not in h:
            continue
        if n:
            out.append(f"| {c} | {fmt_b(b)} | {h['us']:.1f} | {h['busbw']:.1f} | {n['us']:.1f} | "
                       f"{n['busbw']:.1f} | {n['us'] / h['us']:.2f} |")
        else:
            out.append(f"| {c} | {fmt_b(b)} | {h['us']:.1f} | {h['busbw']:.1f} | — | — | — |")
    out.append("")
    extra = []
    for tag, title in (("ar_single", "all-reduce, `single` formulation (one step)"),
                       ("chain", "broadcast / reduce as pipelined chains (g=1, ring=p)"),
                       ("ar_pipe", "all-reduce `multi` with pipelining"),
                       ("nvls", "NVLS windows (multimem), opt-in")):
        rs = rows(d / f"sweep_p{p}_{tag}.jsonl")
        if not rs:
            continue
        extra.append(f"### p = {p}: {title}\n")
        extra.append("| collective | formulation | m | S | µs | busbw GB/s |")
        extra.append("|---|---|---|---|---|---|")
        for r in rs:
            extra.append(f"| {r['collective']} | {r.get('formulation', '')} | {r.get('pipeline')} | "
                         f"{fmt_b(r['bytes'])} | {r.get('us', 0):.1f} | {r.get('busbw', 0):.1f} |")
        extra.append("")
    out += extra
print("\n".join(out))
