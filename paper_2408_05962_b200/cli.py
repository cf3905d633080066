"""Command line over the hiccl host path, mirroring the reference CLI's
subcommands (proj/tools/hiercoll_cli.cpp:184-241) with the B200 cost model
in place of the α-β simulator:

  python -m paper_2408_05962_b200 plan     --collective all_reduce --formulation multi --p 8 --count 1024
  python -m paper_2408_05962_b200 lower    ... [--machine m.toy | --hierarchy 2,4 --gpn 4] --stripe s --ring n
  python -m paper_2408_05962_b200 pipeline ... --pipeline m
  python -m paper_2408_05962_b200 matrix   ... --stage k          (CSV, bytes src -> dst of slot k)
  python -m paper_2408_05962_b200 check    ... [--execs E] [--gpus N]
  python -m paper_2408_05962_b200 simulate ... [--copy-mode push|pull|ll] [--nvls] [--dtype f32]
  python -m paper_2408_05962_b200 sweep    ... --stripe 1,2 --ring 1,2 --pipeline 1,4 --count 256,4096
  python -m paper_2408_05962_b200 bounds   --p 16 [--machine m.toy]
  python -m paper_2408_05962_b200 tune     --collective all_reduce --p 8 --count 33554432 [--nvls]

`check` verifies what the executors would run: the schedule replayed
against the reference's sequential (slot, id) order with an order-sensitive
fold, and every tile hazard of the device layout (CPU, no GPU needed);
with --gpus N it also runs the plan on N GPUs through the C ABI on integer
inputs and compares every rank's buffers with the collective's definition.
Exit codes as the reference: 0 ok, 1 error or FAIL, 2 usage.
`--cache DIR` memoizes lowering on disk (hiccl.PlanCache).
"""
from __future__ import annotations

import argparse
import json
import sys

from . import hiccl as H

KINDS = ["scatter", "broadcast", "gather", "reduce", "all_to_all", "all_gather",
         "reduce_scatter", "all_reduce"]
FORMS = ["single", "multi", "multi_alt"]


def _csv_ints(text: str) -> list[int]:
    try:
        out = [int(x) for x in text.split(",") if x.strip()]
    except ValueError:
        raise H.HicclError(10, f"ParseError: bad integer list '{text}'")
    if not out:
        raise H.HicclError(10, f"ParseError: empty list '{text}'")
    return out


def load_machine(args, p: int) -> tuple[H.Machine, dict]:
    """hiercoll-machine-v1 file (machines/*.toy) or --hierarchy/--gpn flags."""
    if args.machine:
        with open(args.machine) as f:
            m = json.load(f)
        if m.get("format") != "hiercoll-machine-v1":
            raise H.HicclError(10, f"ParseError: {args.machine}: not hiercoll-machine-v1")
        hier = list(m["hierarchy"])
        lib = [lv.get("transport", "") for lv in m.get("levels", [])] or None
        return H.Machine(hier, m.get("gpus_per_node", 0), lib), m
    hier = _csv_ints(args.hierarchy) if args.hierarchy else [p]
    lib = args.library.split(",") if args.library else None
    return H.Machine(hier, args.gpn, lib), {}


def _spec(args) -> H.CollectiveSpec:
    if args.collective not in KINDS:
        raise H.HicclError(10, f"ParseError: unknown collective '{args.collective}'")
    if args.formulation not in FORMS:
        raise H.HicclError(10, f"ParseError: unknown formulation '{args.formulation}'")
    return H.CollectiveSpec(H.CollectiveKind(KINDS.index(args.collective)),
                            H.Formulation(FORMS.index(args.formulation)), args.root,
                            args.count, H.ReduceOp(0 if args.op == "sum" else 1))


def obtain_program(args) -> H.CollectiveProgram:
    if getattr(args, "program", None):
        with open(args.program) as f:
            return H.CollectiveProgram.deserialize(f.read())
    return H.build(_spec(args), args.p)


def obtain_plan(args, pipeline: int | None = None) -> H.Plan:
    prog = obtain_program(args)
    machine, _ = load_machine(args, args.p)
    m = args.pipeline if pipeline is None else pipeline
    if args.cache:
        return H.PlanCache(args.cache).lower(prog, machine, args.ring, args.stripe, m)
    return H.lower(prog, machine, ring=args.ring, stripe=args.stripe, pipeline=m)


def write_out(path: str, text: str) -> None:
    if path:
        with open(path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text if text.endswith("\n") else text + "\n")


def _expected_i32(kind: int, p: int, d: int, root: int, sends, recv_init):
    """The collective's definition on integers (wrapping sums)."""
    import numpy as np
    out = [r.copy() for r in recv_init]

    def red(sl):
        acc = np.stack([s[sl] for s in sends]).astype(np.int64).sum(axis=0)
        return ((acc + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32)

    for j in range(p):
        if kind == 0:
            out[j][:d] = sends[root][j * d:(j + 1) * d]
        elif kind == 1:
            out[j][:p * d] = sends[root][:p * d]
        elif kind == 2 and j == root:
            for i in range(p):
                out[j][i * d:(i + 1) * d] = sends[i][:d]
        elif kind == 3 and j == root:
            out[j][:p * d] = red(slice(0, p * d))
        elif kind == 4:
            for i in range(p):
                out[j][i * d:(i + 1) * d] = sends[i][j * d:(j + 1) * d]
        elif kind == 5:
            for i in range(p):
                out[j][i * d:(i + 1) * d] = sends[i][:d]
        elif kind == 6:
            out[j][j * d:(j + 1) * d] = red(slice(j * d, (j + 1) * d))
        elif kind == 7:
            out[j][:p * d] = red(slice(0, p * d))
    return out


def _run_on_gpus(plan: H.Plan, args) -> tuple[bool, str]:
    import numpy as np
    import torch
    kind = KINDS.index(args.collective)
    p, d = args.p, args.count
    devices = list(range(args.gpus))
    send_len, recv_len = H.preset_lengths(_spec(args), p)
    rng = np.random.default_rng(1234)
    sends = [rng.integers(-2 ** 20, 2 ** 20, send_len, dtype=np.int32) for _ in range(p)]
    recv0 = [np.full(recv_len, -7, dtype=np.int32) for _ in range(p)]
    world = H.World(plan, devices, "i32", copy_mode=args.copy_mode)
    tensors = {}
    try:
        for r in range(p):
            dev = world.device_of(r)
            for name, host in (("sendbuf", sends[r]), ("recvbuf", recv0[r])):
                t = torch.from_numpy(host.copy()).to(f"cuda:{dev}")
                world.bind(r, name, t.data_ptr(), t.numel() * 4)
                tensors[(name, r)] = t
        world.commit()
        world.run()
        for dv in devices:
            torch.cuda.synchronize(dv)
        got = [tensors[("recvbuf", r)].cpu().numpy() for r in range(p)]
    finally:
        world.close()
    want = _expected_i32(kind, p, d, args.root, sends, recv0)
    for r in range(p):
        bad = np.nonzero(got[r] != want[r])[0]
        if bad.size:
            i = int(bad[0])
            return False, (f"rank {r} recvbuf[{i}] = {int(got[r][i])}, expected {int(want[r][i])} "
                           f"({bad.size} elements differ)")
    return True, ""


def cmd_check(args) -> int:
    plan = obtain_plan(args)
    execs = args.execs or min(args.p, 8)
    summ = plan.schedule_summary(num_execs=execs, copy_mode=args.copy_mode, verify=True)
    msg = (f"schedule: {summ['items']} write groups, {summ['steps']} steps, "
           f"{execs} executors, order and hazards verified")
    if args.gpus:
        ok, why = _run_on_gpus(plan, args)
        if not ok:
            print(f"FAIL: {why}")
            return 1
        msg += f"; device run on {args.gpus} GPU(s) matches the collective"
    print(f"PASS ({msg})")
    return 0


def _simulate_row(args, prog_p: int, count: int, s: int, n: int, m: int) -> str:
    spec = _spec(args)
    spec.count = count
    prog = H.build(spec, prog_p)
    machine, _ = load_machine(args, prog_p)
    plan = H.lower(prog, machine, ring=n, stripe=s, pipeline=m)
    esz = H.ELEMENT_SIZE[args.dtype]
    if args.nvls:
        t = H.predict_nvls(plan, args.dtype)
    else:
        t = H.predict(plan, esz, ranks_per_gpu=args.ranks_per_gpu, copy_mode=args.copy_mode)
    S = count * prog_p * esz
    return (f"{args.collective},{args.formulation},{prog_p},{count},{s},{n},{m},"
            f"{args.copy_mode if not args.nvls else 'nvls'},{t:.9g},{S / t / 1e9:.6g}\n")


SIM_HEADER = "collective,formulation,p,count,stripe,ring,pipeline,mode,seconds,algbw_GBps\n"


def main(argv: list[str] | None = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2408_05962_b200",
                                 description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def coll(c):
        c.add_argument("--collective", default="broadcast")
        c.add_argument("--formulation", default="single")
        c.add_argument("--p", type=int, default=4)
        c.add_argument("--count", type=int, default=1024, help="per-rank chunk length d")
        c.add_argument("--root", type=int, default=0)
        c.add_argument("--op", default="sum", choices=["sum", "max"])
        c.add_argument("--out", default="")

    def cfg(c, lists=False):
        c.add_argument("--machine", default="", help="hiercoll-machine-v1 file")
        c.add_argument("--hierarchy", default="", help="e.g. 2,4 (default flat {p})")
        c.add_argument("--gpn", type=int, default=0, help="gpus per node g (default p)")
        c.add_argument("--library", default="", help="per-level transport labels")
        c.add_argument("--program", default="", help="serialized program instead of a preset")
        c.add_argument("--cache", default="", help="plan cache directory")
        typ = str if lists else int
        c.add_argument("--stripe", type=typ, default="1" if lists else 1)
        c.add_argument("--ring", type=typ, default="1" if lists else 1)
        c.add_argument("--pipeline", type=typ, default="1" if lists else 1)

    c = sub.add_parser("plan", help="emit a collective program")
    coll(c)
    c = sub.add_parser("lower", help="lower a program to a staged plan (hiercoll-plan-v1)")
    coll(c), cfg(c)
    c = sub.add_parser("pipeline", help="pipeline a plan into slots (hiercoll-pipelined-v1)")
    coll(c), cfg(c)
    c = sub.add_parser("matrix", help="bytes src -> dst of one slot, CSV")
    coll(c), cfg(c)
    c.add_argument("--stage", type=int, required=True, help="slot index")
    c = sub.add_parser("check", help="verify the executors' schedule (and a device run)")
    coll(c), cfg(c)
    c.add_argument("--execs", type=int, default=0, help="executors (GPUs) the schedule targets")
    c.add_argument("--copy-mode", default="push", choices=["pull", "push", "staged", "ll"])
    c.add_argument("--gpus", type=int, default=0, help="also run on this many GPUs")
    for name in ("simulate", "sweep"):
        c = sub.add_parser(name, help="B200 cost model: one configuration" if name == "simulate"
                           else "B200 cost model over a grid (comma lists)")
        coll(c), cfg(c, lists=name == "sweep")
        c.add_argument("--copy-mode", default="push", choices=["pull", "push", "staged", "ll"])
        c.add_argument("--nvls", action="store_true", help="user buffers in an NVLS window")
        c.add_argument("--dtype", default="f32")
        c.add_argument("--ranks-per-gpu", type=int, default=1)
        if name == "sweep":
            c.add_argument("--counts", default="", help="comma list of d (default --count)")
    c = sub.add_parser("bounds", help="Table-4 asymptotic throughput limits (CSV)")
    c.add_argument("--p", type=int, required=True)
    c.add_argument("--machine", default="")
    c.add_argument("--gpn", type=int, default=0)
    c.add_argument("--hierarchy", default="")
    c.add_argument("--library", default="")
    c.add_argument("--nics", type=int, default=1)
    c.add_argument("--nic-bandwidth", type=float, default=25e9)
    c.add_argument("--out", default="")
    c = sub.add_parser("tune", help="cost-model choice of formulation / ring / pipeline / mode")
    coll(c)
    c.add_argument("--dtype", default="f32")
    c.add_argument("--nvls", action="store_true", help="also weigh the NVLS library")

    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if args.cmd == "plan":
            write_out(args.out, obtain_program(args).serialize())
        elif args.cmd == "lower":
            prog = obtain_program(args)
            machine, _ = load_machine(args, args.p)
            write_out(args.out, H.lower_staged_json(prog, machine, ring=args.ring, stripe=args.stripe))
        elif args.cmd == "pipeline":
            write_out(args.out, obtain_plan(args).serialize())
        elif args.cmd == "matrix":
            plan = obtain_plan(args)
            if not 0 <= args.stage < plan.slots:
                raise H.HicclError(9, f"InvalidConfig: --stage {args.stage} outside schedule of "
                                      f"{plan.slots} slots")
            rows = plan.comm_matrix(args.stage)  # bytes at the machine's element size (4)
            write_out(args.out, "".join(",".join(str(v) for v in r) + "\n" for r in rows))
        elif args.cmd == "check":
            return cmd_check(args)
        elif args.cmd == "simulate":
            write_out(args.out, SIM_HEADER + _simulate_row(args, args.p, args.count, args.stripe,
                                                           args.ring, args.pipeline))
        elif args.cmd == "sweep":
            counts = _csv_ints(args.counts) if args.counts else [args.count]
            text = SIM_HEADER
            for d in counts:
                for s in _csv_ints(args.stripe):
                    for n in _csv_ints(args.ring):
                        for m in _csv_ints(args.pipeline):
                            text += _simulate_row(args, args.p, d, s, n, m)
            write_out(args.out, text)
        elif args.cmd == "bounds":
            g, k, f = args.gpn or args.p, args.nics, args.nic_bandwidth
            if args.machine:
                with open(args.machine) as fh:
                    m = json.load(fh)
                g, k, f = m.get("gpus_per_node", g), m.get("nics_per_node", k), m.get("nic_bandwidth", f)
            text = "collective,p,g,k,f_Bps,bound_Bps,bound_GBps\n"
            for i, name in enumerate(KINDS):
                b = H.bound(H.CollectiveKind(i), args.p, g, k, f)
                text += f"{name},{args.p},{g},{k},{f:.6g},{b:.6g},{b / 1e9:.6g}\n"
            write_out(args.out, text)
        elif args.cmd == "tune":
            kind = H.CollectiveKind(KINDS.index(args.collective))
            if args.nvls:
                t = H.tune_nvls(kind, args.p, args.count, args.dtype)
            else:
                t = H.tune(kind, args.p, args.count, H.ELEMENT_SIZE[args.dtype])
            t["formulation"] = FORMS[int(t["formulation"])]
            write_out(args.out, json.dumps(t))
        return 0
    except (H.HicclError, OSError, ValueError, KeyError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
