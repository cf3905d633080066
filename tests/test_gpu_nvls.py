"""NVLS lowering (per-level library "NVLS"): user buffers in a multicast
window, reduction groups over every rank reduced inside the NVSwitch
(multimem.ld_reduce), multicasts to every rank written once (multimem.st).

Copies and integer reductions stay bit-exact (checked against the oracle);
floating-point sums are reduced in the switch's order (fp32 accumulation
for 16-bit types), so they are checked against the exact sum of the inputs
(fp64) within the stated tolerance: |got - exact| <= rtol * sum_i |x_i|,
rtol 1e-6 (f32) and 1e-2 (bf16, f16)."""
import numpy as np
import pytest

import oracle
from tests import harness

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
REF = oracle.Reference() if oracle.reference_available() else None
RTOL = {"f32": 1e-6, "bf16": 1e-2, "f16": 1e-2}


def devices():
    import torch
    n = torch.cuda.device_count()
    return tuple(range(4 if n >= 4 else 2))


def nvls_ok():
    from paper_2408_05962_b200 import hiccl as H
    return H.nvls_supported(0)


@pytest.mark.parametrize("kind,form,dtype", [(7, 1, "f32"), (7, 1, "bf16"), (7, 0, "f32"),
                                             (6, 0, "f32"), (5, 0, "f32"), (7, 1, "i32"),
                                             (5, 0, "bf16"), (7, 2, "f32")])
def test_nvls_collectives(kind, form, dtype):
    if not nvls_ok():
        pytest.skip("no NVSwitch multicast")
    devs = devices()
    p = len(devs)
    d = 1 << 16
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 1)
    flat = harness.oracle_plan(plan, kind, form, p, d, 0, 0, [p], p, 1, 1, 1, REF)
    want = harness.run_oracle(flat, plan, dtype, 77)
    got, stats = harness.run_device(plan, dtype, 77, devices=devs, nvls=True)
    assert sum(s["nvls_items"] for s in stats) > 0, stats
    if dtype in RTOL and kind in (3, 6, 7):
        st = harness.initial_state(plan, dtype, 77)
        exact = harness.exact_reduction(kind, p, d, 0, dtype, st["sendbuf"], st["recvbuf"])
        harness.assert_close(got, exact, dtype, st["sendbuf"], RTOL[dtype],
                             f"nvls {kind}/{form} {dtype}")
    else:
        harness.assert_bitwise(got, want, f"nvls {kind}/{form} {dtype}")


def test_nvls_unlowerable_items_keep_p2p():
    # all-to-all has no every-rank group: nothing lowered, results exact
    if not nvls_ok():
        pytest.skip("no NVSwitch multicast")
    devs = devices()
    p = len(devs)
    plan, _, _ = harness.make_plan(4, 0, p, 4096, 0, 0, [p], p, 1, 1, 1)
    flat = harness.oracle_plan(plan, 4, 0, p, 4096, 0, 0, [p], p, 1, 1, 1, REF)
    want = harness.run_oracle(flat, plan, "f32", 5)
    got, stats = harness.run_device(plan, "f32", 5, devices=devs, nvls=True)
    assert all(s["nvls_items"] == 0 for s in stats)
    harness.assert_bitwise(got, want, "a2a nvls window")


@pytest.mark.parametrize("dtype,m", [("f32", 1), ("f32", 4), ("bf16", 2), ("i32", 4)])
def test_nvls_fused_all_reduce(dtype, m):
    # all-reduce multi with both buffers in the window: every reduce-scatter
    # group and its in-place all-gather multicast fuse into one
    # reduce+multicast item per pipeline channel (layout.hpp fuse_nvls)
    if not nvls_ok():
        pytest.skip("no NVSwitch multicast")
    devs = devices()
    p = len(devs)
    d = 3 << 14
    plan, _, _ = harness.make_plan(7, 1, p, d, 0, 0, [p], p, 1, 1, m)
    summ = plan.layout_summary(num_execs=p, rank_to_exec=list(range(p)), dtype=dtype,
                               multicast=["sendbuf", "recvbuf"])
    assert summ["fused"] == p * m
    got, stats = harness.run_device(plan, dtype, 91, devices=devs, nvls=True)
    assert all(s["nvls_items"] == m for s in stats), stats
    if dtype == "i32":  # integer sums are order-free: bit-exact vs the oracle
        flat = harness.oracle_plan(plan, 7, 1, p, d, 0, 0, [p], p, 1, 1, m, REF)
        harness.assert_bitwise(got, harness.run_oracle(flat, plan, dtype, 91), "fused i32")
    else:
        st = harness.initial_state(plan, dtype, 91)
        exact = harness.exact_reduction(7, p, d, 0, dtype, st["sendbuf"], st["recvbuf"])
        harness.assert_close(got, exact, dtype, st["sendbuf"], RTOL[dtype], f"fused {dtype} m={m}")
    # every rank holds the same bits (one reduction, multicast to all)
    for r in range(1, p):
        assert (got["recvbuf"][r].view("u1") == got["recvbuf"][0].view("u1")).all()


@pytest.mark.parametrize("kind,form", [(7, 1), (7, 2), (5, 0), (6, 0)])
@pytest.mark.parametrize("dtype", ["f32", "i32"])
def test_nvls_back_to_back_epochs(kind, form, dtype):
    """12 launches back to back with the buffers in the NVLS window: between
    launches every rank's inputs are rewritten on its executor's stream and
    every output is snapshotted, no host synchronization. A multicast write
    of epoch e not ordered before a peer's unicast read (or the reverse —
    the two aliases of one physical buffer, fence.proxy.alias at every flag
    hand-off) would corrupt a snapshot. i32: bit-exact against the oracle
    per epoch; f32: within rtol of the exact sum (switch order)."""
    import torch
    from paper_2408_05962_b200 import hiccl as H
    if not nvls_ok():
        pytest.skip("no NVSwitch multicast")
    devs = devices()
    p = len(devs)
    d, epochs = 1 << 14, 12
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 1)
    world = H.World(plan, devs, dtype, copy_mode="push")
    esz = H.ELEMENT_SIZE[dtype]
    try:
        sizes = {name: length * esz for name, length, inp, internal in plan.buffers if not internal}
        where = world.enable_nvls(sizes)
        world.commit()
        assert sum(e.stats()["nvls_items"] for e in world.execs) > 0
        streams = [torch.cuda.Stream(dv) for dv in devs]
        views = {k: torch.as_tensor(H.DeviceView(v, sizes[k[1]]), device=f"cuda:{world.device_of(k[0])}")
                 for k, v in where.items()}
        for k, t in views.items():
            with torch.cuda.stream(streams[world.rank_to_exec[k[0]]]):
                t.zero_()
        snaps = {}
        inputs = {name for name, length, inp, internal in plan.buffers if inp and not internal}
        for e in range(epochs):
            for (r, name), ptr in where.items():
                if name in inputs:
                    x = world.rank_to_exec[r]
                    H.device_fill(devs[x], ptr, sizes[name] // esz, dtype, 500 + e, r,
                                  stream=streams[x].cuda_stream)
            for i, ex in enumerate(world.execs):
                ex.start(streams[i].cuda_stream)
            for (r, name), t in views.items():
                if name not in inputs:
                    with torch.cuda.stream(streams[world.rank_to_exec[r]]):
                        snaps[(e, r, name)] = t.clone()
        world.wait()
        for dv in set(devs):
            torch.cuda.synchronize(dv)
        flat = harness.oracle_plan(plan, kind, form, p, d, 0, 0, [p], p, 1, 1, 1, REF)
        prev = None
        for e in range(epochs):
            st = {}
            for name, length, inp, internal in plan.buffers:
                if internal:
                    continue
                st[name] = [oracle.fill(length, dtype, 500 + e, r) if inp else
                            (np.zeros(length, oracle.DTYPES[dtype][1]) if prev is None
                             else prev[name][r].copy()) for r in range(p)]
            sends = [a.copy() for a in st["sendbuf"]]
            recv0 = [a.copy() for a in st["recvbuf"]]
            oracle.execute(flat, dtype, st)
            got = {"recvbuf": [snaps[(e, r, "recvbuf")].cpu().numpy().view(st["recvbuf"][r].dtype)
                               for r in range(p)]}
            if dtype == "i32" or kind == 5:
                harness.assert_bitwise(got, {"recvbuf": st["recvbuf"]}, f"epoch {e}")
            else:
                exact = harness.exact_reduction(kind, p, d, 0, dtype, sends, recv0)
                harness.assert_close(got, exact, dtype, sends, RTOL[dtype], f"epoch {e}")
            prev = {"recvbuf": got["recvbuf"], "sendbuf": st["sendbuf"]}
    finally:
        world.close()


def test_nvls_checked_mode(monkeypatch):
    """HICCL_CHECK_DEPS=1 on multimem launches: every producer flag is
    re-read before each step (the fused reduce+multicast and a pipelined
    all-reduce); results stay within tolerance / bit-exact."""
    if not nvls_ok():
        pytest.skip("no NVSwitch multicast")
    monkeypatch.setenv("HICCL_CHECK_DEPS", "1")
    devs = devices()
    p = len(devs)
    for kind, form, m, dtype in [(7, 1, 1, "i32"), (7, 1, 3, "i32"), (5, 0, 2, "f32")]:
        d = 3 << 13
        plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, m)
        flat = harness.oracle_plan(plan, kind, form, p, d, 0, 0, [p], p, 1, 1, m, REF)
        want = harness.run_oracle(flat, plan, dtype, 13)
        got, stats = harness.run_device(plan, dtype, 13, devices=devs, nvls=True)
        assert sum(s["nvls_items"] for s in stats) > 0
        harness.assert_bitwise(got, want, f"checked nvls {kind}/{form} m={m} {dtype}")
