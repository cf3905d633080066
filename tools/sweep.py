#!/usr/bin/env python
"""Message-size sweep of all eight collectives, hiccl vs NCCL, one process
per GPU (torchrun). Writes one JSON line per (collective, size, impl) to
stdout and, with --out, to a file (profiles/ keeps the committed ones).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/sweep.py \
      --sizes 1K,1M,64M,1G --collectives all_reduce,all_gather --out profiles/sweep_p4.jsonl

Size S is the per-rank buffer in bytes as in SURVEY §8(d): sendbuf for
AR/RS/Bcast/Reduce/A2A, recvbuf for AG/Gather, the root's sendbuf for
Scatter. algbw = S / t, busbw = algbw * F (2(p-1)/p AR; (p-1)/p AG, RS, A2A,
Scatter, Gather; 1 Bcast, Reduce). t = max over ranks of the mean CUDA-event
time of `--iters` back-to-back executions after `--warmup`.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

KINDS = ["scatter", "broadcast", "gather", "reduce", "all_to_all", "all_gather",
         "reduce_scatter", "all_reduce"]
FORM = {"scatter": 0, "broadcast": 1, "gather": 0, "reduce": 1, "all_to_all": 0, "all_gather": 0,
        "reduce_scatter": 0, "all_reduce": 1}


def parse_size(s: str) -> int:
    s = s.strip().upper()
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(float(s[:-1]) * mult[s[-1]]) if s[-1] in mult else int(s)


def busbw_factor(kind: str, p: int) -> float:
    if p == 1:
        return 1.0
    if kind == "all_reduce":
        return 2 * (p - 1) / p
    if kind in ("broadcast", "reduce"):
        return 1.0
    return (p - 1) / p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1K,64K,1M,16M,256M,1G")
    ap.add_argument("--collectives", default=",".join(KINDS))
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--pipeline", type=int, default=1)
    ap.add_argument("--copy-mode", default="push")
    ap.add_argument("--formulation", default="", help="override, e.g. single")
    ap.add_argument("--hierarchy", default="", help="e.g. 2,2 (default flat {p})")
    ap.add_argument("--gpn", type=int, default=0, help="gpus_per_node g for the plan (default p)")
    ap.add_argument("--stripe", type=int, default=1)
    ap.add_argument("--ring", type=int, default=1)
    ap.add_argument("--nccl", action="store_true")
    ap.add_argument("--out", default="")
    ap.add_argument("--trace", action="store_true", help="add the device timeline of the last launch")
    ap.add_argument("--ranks-per-gpu", type=int, default=1, help="logical ranks per GPU (virtual p)")
    ap.add_argument("--root", type=int, default=0)
    ap.add_argument("--nvls", action="store_true", help="buffers in an NVLS window (multimem)")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--auto", action="store_true",
                    help="per size, the cost model's formulation / ring / pipeline / copy mode")
    ap.add_argument("--graph", action="store_true",
                    help="capture the --iters launches in a CUDA graph and time its replay "
                         "(device-side latency without host launch cost; NCCL likewise)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2408_05962_b200 import hiccl as H
    from paper_2408_05962_b200.dist import DistCommunicator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    dev = local
    p = world * args.ranks_per_gpu
    esz = H.ELEMENT_SIZE[args.dtype]
    hier = [int(x) for x in args.hierarchy.split(",")] if args.hierarchy else [p]
    g = args.gpn or p
    stream = torch.cuda.Stream(dev)
    out_f = open(args.out, "a") if (args.out and rank == 0) else None

    def allgather(obj):
        if world == 1:
            return [obj]
        o = [None] * world
        dist.all_gather_object(o, obj)
        return o

    def tmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()

    def emit(rec):
        if rank == 0:
            line = json.dumps(rec)
            print(line, flush=True)
            if out_f:
                out_f.write(line + "\n")
                out_f.flush()

    ng = dist.new_group(backend="nccl") if (args.nccl and world > 1) else None

    for kind_name in args.collectives.split(","):
        kind = KINDS.index(kind_name)
        form = FORM[kind_name]
        if args.formulation:
            form = {"single": 0, "multi": 1, "multi_alt": 2}[args.formulation]
        if kind in (0, 2, 4):
            form = 0
        for size_s in args.sizes.split(","):
            S = parse_size(size_s)
            d = max(1, S // (esz * p)) if kind not in (2, 5) else max(1, S // (esz * p))
            root = args.root if kind in (0, 1, 2, 3) else 0
            ring, pipe, mode, gg, f = args.ring, args.pipeline, args.copy_mode, g, form
            use_nvls = args.nvls
            if args.auto:  # the cost model's choice (H.tune / H.tune_nvls) for this size
                if args.nvls and args.ranks_per_gpu == 1:
                    t = H.tune_nvls(H.CollectiveKind(kind), p, d, args.dtype)
                    use_nvls = t["nvls"]
                else:
                    t = H.tune(H.CollectiveKind(kind), p, d, esz)
                f, ring, pipe, mode = int(t["formulation"]), t["ring"], t["pipeline"], t["copy_mode"]
                gg = 1 if ring > 1 else p
            spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(f), root, d)
            send_len, recv_len = H.preset_lengths(spec, p)
            S_eff = d * p * esz
            try:
                plan = H.lower(H.build(spec, p), H.Machine(hier, gg), ring=ring,
                               stripe=args.stripe, pipeline=pipe)
                comm = DistCommunicator(plan, rank, world, dev, args.dtype,
                                        copy_mode=mode, timeout_s=60.0,
                                        ctas=args.ctas, threads=args.threads)
            except H.HicclError as e:
                emit({"collective": kind_name, "bytes": S_eff, "p": p, "impl": "hiccl",
                      "error": str(e)})
                continue
            bufs = {}
            if use_nvls:
                where = comm.enable_nvls({"sendbuf": send_len * esz, "recvbuf": recv_len * esz},
                                         allgather)
                r = comm.local_ranks[0]
                H.device_fill(dev, where["sendbuf"], send_len, args.dtype, 1234, r)
            else:
                for r in comm.local_ranks:
                    send = torch.empty(send_len * esz, dtype=torch.uint8, device=dev)
                    recv = torch.zeros(recv_len * esz, dtype=torch.uint8, device=dev)
                    H.device_fill(dev, send.data_ptr(), send_len, args.dtype, 1234, r)
                    comm.register(r, "sendbuf", send.data_ptr(), send.numel())
                    comm.register(r, "recvbuf", recv.data_ptr(), recv.numel())
                    bufs[r] = (send, recv)
            comm.connect(allgather)
            sp = stream.cuda_stream
            for _ in range(args.warmup):
                comm.start(sp)
            comm.wait()
            torch.cuda.synchronize(dev)
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            if args.graph:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=stream):
                    for _ in range(args.iters):
                        comm.start(sp)
                with torch.cuda.stream(stream):
                    graph.replay()
                torch.cuda.synchronize(dev)
                barrier()
                with torch.cuda.stream(stream):
                    a.record(stream)
                    graph.replay()
                    b.record(stream)
            else:
                a.record(stream)
                for _ in range(args.iters):
                    comm.start(sp)
                b.record(stream)
            comm.wait()
            torch.cuda.synchronize(dev)
            t = tmax(a.elapsed_time(b) / 1e3 / args.iters)
            alg = S_eff / t / 1e9
            st = comm.executor.stats()
            trace = allgather(comm.executor.trace()) if args.trace else None
            emit({"trace": trace, "collective": kind_name, "formulation": ["single", "multi", "multi_alt"][f],
                  "bytes": S_eff, "p": p, "impl": "hiccl", "dtype": args.dtype,
                  "hierarchy": hier, "g": gg, "stripe": args.stripe, "ring": ring,
                  "pipeline": pipe, "copy_mode": ["pull", "push", "staged", "ll"][st["copy_mode"]],
                  "auto": args.auto, "ctas": st["ctas"], "us": t * 1e6,
                  "algbw": alg, "busbw": alg * busbw_factor(kind_name, p),
                  "steps": st["num_steps"], "items": st["num_items"],
                  "nvls_items": st["nvls_items"], "nvls": use_nvls, "graph": args.graph})
            comm.close()
            del bufs
            barrier()

            if ng is not None and kind_name in ("all_reduce", "all_gather", "reduce_scatter",
                                                "broadcast", "reduce", "all_to_all"):
                tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16,
                       "i32": torch.int32, "i64": torch.int64, "f64": torch.float64,
                       "u8": torch.uint8}[args.dtype]
                x = torch.ones(send_len, dtype=tdt, device=dev)
                y = torch.empty(recv_len, dtype=tdt, device=dev)

                def op():
                    if kind_name == "all_reduce":
                        dist.all_reduce(x, group=ng)
                    elif kind_name == "all_gather":
                        dist.all_gather_into_tensor(y, x, group=ng)
                    elif kind_name == "reduce_scatter":
                        dist.reduce_scatter_tensor(y[:d], x, group=ng)
                    elif kind_name == "broadcast":
                        dist.broadcast(x, 0, group=ng)
                    elif kind_name == "reduce":
                        dist.reduce(x, 0, group=ng)
                    else:
                        dist.all_to_all_single(y, x, group=ng)
                for _ in range(args.warmup):
                    op()
                torch.cuda.synchronize(dev)
                barrier()
                if args.graph:
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph, stream=stream):
                        for _ in range(args.iters):
                            op()
                    with torch.cuda.stream(stream):
                        graph.replay()
                    torch.cuda.synchronize(dev)
                    barrier()
                    with torch.cuda.stream(stream):
                        a.record(stream)
                        graph.replay()
                        b.record(stream)
                else:
                    a.record()
                    for _ in range(args.iters):
                        op()
                    b.record()
                torch.cuda.synchronize(dev)
                t = tmax(a.elapsed_time(b) / 1e3 / args.iters)
                alg = S_eff / t / 1e9
                emit({"collective": kind_name, "bytes": S_eff, "p": p, "impl": "nccl", "dtype": args.dtype,
                      "us": t * 1e6, "algbw": alg, "busbw": alg * busbw_factor(kind_name, p),
                      "nccl": ".".join(map(str, torch.cuda.nccl.version())), "graph": args.graph})
                del x, y
                barrier()
    if out_f:
        out_f.close()
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
