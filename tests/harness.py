"""Shared parity harness: build a preset collective, run it through the
product (libhiccl.so executor on the GPU) and through the oracle
(numeric restatement of the reference executor on the reference's own
plan when oracle/_ref is built, else on the product plan), compare.

Used by tests/ and __graft_entry__.smoke(); the oracle is only the checker.
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_2408_05962_b200 import hiccl as H

SEEDS = (1234, 0xC0FFEE)


def make_plan(kind: int, form: int, p: int, d: int, root: int = 0, op: int = 0,
              hier=None, g: int | None = None, ring: int = 1, stripe: int = 1,
              pipeline: int = 1, library=None):
    hier = list(hier) if hier else [p]
    spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), root, d, H.ReduceOp(op))
    prog = H.build(spec, p)
    machine = H.Machine(hier, g or p, library)
    plan = H.lower(prog, machine, ring=ring, stripe=stripe, pipeline=pipeline)
    return plan, spec, prog


def gpus(n: int) -> tuple:
    """Devices for n executors: n distinct GPUs when the box has them, else
    executors sharing the available ones round robin (each on its own stream
    with 1/k of the device's CTAs; the cross-executor protocol — entry/exit
    barriers, system-scope step flags, peer loads and stores, tagged lines —
    is the same as between GPUs, only the link is HBM instead of NVLink)."""
    import torch
    k = torch.cuda.device_count()
    return tuple(range(n)) if k >= n else tuple(i % k for i in range(n))


def initial_state(plan: H.Plan, dtype: str, seed: int) -> dict[str, list[np.ndarray]]:
    """Inputs from the shared generator; every other user buffer gets the
    sentinel pattern so unwritten elements are caught."""
    st = {}
    for name, length, inp, internal in plan.buffers:
        if internal:
            continue
        st[name] = [oracle.fill(length, dtype, seed, r) if inp else oracle.sentinel(length, dtype, r)
                    for r in range(plan.world_size)]
    return st


def oracle_plan(plan: H.Plan, kind: int, form: int, p: int, d: int, root: int, op: int, hier,
                g, ring, stripe, pipeline, ref: "oracle.Reference | None" = None):
    """The reference's own plan when the reference library is built."""
    if ref is not None:
        rc, text = ref.preset_plan(kind, form, p, d, root, op, list(hier), g, stripe, ring,
                                   pipeline)
        if rc == 0:
            return oracle.FlatPlan.from_json(text)
    return oracle.FlatPlan.from_dicts(plan.world_size, plan.buffers, plan.transfer_dicts())


def run_oracle(flat: oracle.FlatPlan, plan: H.Plan, dtype: str, seed: int, threads: int = 1):
    st = initial_state(plan, dtype, seed)
    oracle.execute(flat, dtype, st, threads=threads)
    return {k: v for k, v in st.items() if k in {b[0] for b in plan.buffers if not b[3]}}


def run_device(plan: H.Plan, dtype: str, seed: int, devices=(0,), repeat: int = 1,
               rank_to_exec=None, nvls: bool = False, misalign=None, **exec_kw):
    """Execute on the GPU(s) through the C ABI. Returns final user buffers.
    nvls=True places the user buffers in an NVLS window (one rank per GPU).
    misalign(rank, name) -> bytes: bind each user buffer that many bytes
    into a larger allocation (unaligned user pointers)."""
    import torch
    esz = H.ELEMENT_SIZE[dtype]
    world = H.World(plan, devices, dtype, rank_to_exec=rank_to_exec, **exec_kw)
    init = initial_state(plan, dtype, seed)
    tensors = {}
    try:
        if nvls:
            where = world.enable_nvls({name: per_rank[0].nbytes for name, per_rank in init.items()})
        for name, per_rank in init.items():
            for r, host in enumerate(per_rank):
                dev = world.device_of(r)
                if nvls:
                    t = torch.as_tensor(H.DeviceView(where[(r, name)], host.nbytes),
                                        device=f"cuda:{dev}")
                    t.copy_(torch.from_numpy(host.view(np.uint8).copy()))
                elif misalign is not None:
                    off = misalign(r, name)
                    raw = torch.zeros(host.nbytes + 64, dtype=torch.uint8, device=f"cuda:{dev}")
                    t = raw[off: off + host.nbytes]
                    t.copy_(torch.from_numpy(host.view(np.uint8).copy()))
                    world.bind(r, name, t.data_ptr(), t.numel())
                else:
                    t = torch.from_numpy(host.view(np.uint8).copy()).to(f"cuda:{dev}")
                    world.bind(r, name, t.data_ptr(), t.numel())
                tensors[(name, r)] = t
        world.commit()
        for _ in range(repeat):
            if repeat > 1:  # re-seed the inputs so every round recomputes
                for (name, r), t in tensors.items():
                    t.copy_(torch.from_numpy(init[name][r].view(np.uint8)).to(t.device))
                for d in set(devices):
                    torch.cuda.synchronize(d)
            world.run()
        for d in set(devices):
            torch.cuda.synchronize(d)
        out = {}
        for name, per_rank in init.items():
            out[name] = [tensors[(name, r)].cpu().numpy().view(per_rank[r].dtype)
                         for r in range(plan.world_size)]
        stats = [e.stats() for e in world.execs]
        return out, stats
    finally:
        world.close()


def to_f64(a: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if dtype == "f16":
        return a.view(np.float16).astype(np.float64)
    return a.astype(np.float64)


def exact_reduction(kind: int, p: int, d: int, root: int, dtype: str, sends, recv_init) -> dict:
    """Collective result with the sums computed exactly (fp64), as float64
    arrays; untouched recvbuf elements keep their initial values."""
    sf = [to_f64(s, dtype) for s in sends]
    out = oracle.ground_truth(kind, p, d, root, 0, "f64", sf, [to_f64(r, dtype) for r in recv_init])
    return {"recvbuf": out}


def assert_close(got: dict, want: dict, dtype: str, sends, rtol: float, what: str = ""):
    """|got - want| <= rtol * sum_i |send_i| elementwise (SURVEY §8(c)
    fallback tolerance, relative to the sum of magnitudes)."""
    f64 = lambda a: a if a.dtype == np.float64 else to_f64(a, dtype)
    mag = np.sum([np.abs(to_f64(s, dtype)) for s in sends], axis=0)
    for name in want:
        for r, (g, w) in enumerate(zip(got[name], want[name])):
            n = min(g.size, mag.size)
            err = np.abs(f64(g[:n]) - f64(w[:n]))
            bad = err > rtol * np.maximum(mag[:n], 1e-30)
            assert not bad.any(), f"{what}: {name}@rank{r}: {bad.sum()} elements beyond rtol {rtol}"
            if g.size > n:
                assert (f64(g[n:]) == f64(w[n:])).all(), f"{what}: {name}@rank{r} tail differs"


def assert_bitwise(got: dict, want: dict, what: str = ""):
    for name in want:
        for r, (g, w) in enumerate(zip(got[name], want[name])):
            if g.tobytes() != w.tobytes():
                bad = np.nonzero(g.view(np.uint8) != w.view(np.uint8))[0]
                raise AssertionError(
                    f"{what}: {name}@rank{r} differs in {bad.size} bytes, first at byte {bad[0]}: "
                    f"got {g[bad[0] // g.itemsize]} want {w[bad[0] // w.itemsize]}")
