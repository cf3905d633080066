"""NVLS device layout on CPU (csrc/host/layout.cpp build_layout + fuse_nvls).

With user buffers in an NVSwitch multicast window, every-rank reductions
lower to multimem.ld_reduce and in-place every-rank multicasts to
multimem.st. fuse_nvls then joins a reduction with the later multicast of
its own result (all-reduce = reduce-scatter . all-gather, presets.cpp:208-216)
into one reduce+multicast item per tile. hc_plan_layout_summary runs the
executors' layout and verify_sync (every conflicting tile pair ordered),
so a fusion that broke an ordering would raise DependencyViolation.
"""
import pytest

from paper_2408_05962_b200 import hiccl as H
from tests import harness

MC = ["sendbuf", "recvbuf"]


def kinds(summary, exec_):
    return [k for step in summary["execs"][exec_]["steps"] for k in step]


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_all_reduce_multi_fuses(p, m, dtype):
    plan, _, _ = harness.make_plan(7, 1, p, 1 << 14, pipeline=m)
    s = plan.layout_summary(num_execs=p, rank_to_exec=list(range(p)), dtype=dtype, multicast=MC)
    assert s["fused"] == p * m
    for e in range(p):
        assert kinds(s, e) == ["mc_reduce_store"] * m


def test_no_window_no_lowering():
    plan, _, _ = harness.make_plan(7, 1, 4, 1 << 14)
    s = plan.layout_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3])
    assert s["fused"] == 0
    assert set(kinds(s, 0)) == {"p2p"}


def test_max_f32_not_lowered():
    # the switch has no f32 max: the reduction groups stay point to point,
    # only the all-gather half becomes multimem.st, nothing fuses
    plan, _, _ = harness.make_plan(7, 1, 4, 1 << 14, op=1)
    s = plan.layout_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], multicast=MC)
    assert s["fused"] == 0 and set(kinds(s, 0)) == {"p2p", "mc_store"}


def test_reduce_scatter_and_all_gather_stay_separate():
    for kind in (5, 6):
        plan, _, _ = harness.make_plan(kind, 0, 4, 1 << 14)
        s = plan.layout_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], multicast=MC)
        assert s["fused"] == 0
        assert "mc_reduce_store" not in kinds(s, 0)


def test_virtual_ranks_disable_nvls():
    plan, _, _ = harness.make_plan(7, 1, 8, 1 << 14)
    s = plan.layout_summary(num_execs=4, rank_to_exec=[0, 0, 1, 1, 2, 2, 3, 3], multicast=MC)
    assert s["fused"] == 0 and set(kinds(s, 0)) == {"p2p"}


def _program(p, n, reader_between):
    prog = H.CollectiveProgram(p)
    prog.declare_buffer("sendbuf", n, input=True)
    prog.declare_buffer("recvbuf", n)
    prog.declare_buffer("other", n)
    R = H.BufferRef
    # step 0: rank 0's recvbuf = sum of every rank's sendbuf
    prog.add_reduction(R("sendbuf", 0, n), R("recvbuf", 0, n), list(range(p)), 0)
    prog.add_fence()
    if reader_between:
        # step 1: rank 1 writes its own recvbuf range and copies it away;
        # a fused multicast at step 0 would land before these
        prog.add_multicast(R("sendbuf", 0, n), R("recvbuf", 0, n), 1, [1])
        prog.add_fence()
        prog.add_multicast(R("recvbuf", 0, n), R("other", 0, n), 1, [1])
        prog.add_fence()
    # last step: rank 0 multicasts the result in place to everyone
    prog.add_multicast(R("recvbuf", 0, n), R("recvbuf", 0, n), 0, list(range(1, p)))
    return prog


@pytest.mark.parametrize("reader_between", [False, True])
def test_fusion_only_when_range_is_quiet(reader_between):
    p, n = 4, 1 << 12
    plan = H.lower(_program(p, n, reader_between), H.Machine([p], p))
    s = plan.layout_summary(num_execs=p, rank_to_exec=list(range(p)), multicast=MC)
    if reader_between:
        assert s["fused"] == 0
        assert "mc_reduce" in kinds(s, 0) and "mc_store" in kinds(s, 0)
    else:
        assert s["fused"] == 1
        assert kinds(s, 0) == ["mc_reduce_store"]


@pytest.mark.parametrize("kind,form,m", [(3, 0, 8), (1, 0, 8), (7, 1, 4), (6, 1, 2), (5, 0, 1)])
def test_alternating_halves_keep_every_hazard_ordered(monkeypatch, kind, form, m):
    # consecutive steps on disjoint halves of the grid: the tile hazard
    # check (verify_sync) still finds a wait for every conflicting pair
    monkeypatch.setenv("HICCL_ALT_HALVES", "1")
    hier, g, ring = ([4], 1, 4) if kind in (1, 3) else ([4], 4, 1)
    plan, _, _ = harness.make_plan(kind, form, 4, 1 << 16, 0, 0, hier, g, ring, 1, m)
    s = plan.layout_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], ctas=148)
    assert s["ctas"] == 148


def test_alt_halves_default_only_for_small_pipelined_steps(monkeypatch):
    monkeypatch.delenv("HICCL_ALT_HALVES", raising=False)
    want = {(32 << 20, 8): True, (128 << 20, 8): False, (32 << 20, 1): False}
    for (S, m), on in want.items():
        plan, _, _ = harness.make_plan(3, 0, 4, S // 16, 0, 0, [4], 1, 4, 1, m)
        s = plan.layout_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], ctas=148)
        assert s["alt_halves"] == on, (S, m)
    plan, _, _ = harness.make_plan(7, 1, 4, 1 << 24)  # two big steps
    assert not plan.layout_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3])["alt_halves"]
