"""The executor schedule (csrc/host/schedule.cpp) on CPU.

For every plan the device would run, the schedule must (a) fuse each
slot's writes into write groups whose fold order is the reference's id
order, (b) leave no cross-step RAW/WAR/WAW hazard without a wait edge.
hc_plan_schedule_summary(verify=1) replays the schedule against the
reference's sequential (slot, id) execution with an order-sensitive fold
and checks every hazard pair independently; it raises on any mismatch.
"""
import pytest

from paper_2408_05962_b200 import hiccl as H
from tests import harness

FORMS = [(k, f) for k, fs in {0: [0], 1: [0, 1], 2: [0], 3: [0, 1], 4: [0], 5: [0, 1],
                              6: [0, 1], 7: [0, 1, 2]}.items() for f in fs]
MACHINES = [([8], 8, 1, 1, 1), ([8], 8, 1, 1, 4), ([2, 4], 4, 4, 2, 3), ([2, 4], 4, 1, 1, 16),
            ([2, 2, 2], 2, 2, 4, 2), ([2, 2, 2], 8, 1, 1, 5), ([2, 2, 2], 1, 1, 8, 4),
            ([4, 2], 2, 2, 2, 3)]


@pytest.mark.parametrize("kind,form", FORMS)
@pytest.mark.parametrize("mapping", ["one", "two", "four", "eight-push", "four-staged", "four-ll"])
def test_schedule_replays_reference_order(kind, form, mapping):
    for hier, g, s, n, m in MACHINES:
        plan, _, _ = harness.make_plan(kind, form, 8, 11, 3 if kind < 4 else 0, 0, hier, g, n, s, m)
        execs = {"one": 1, "two": 2, "four": 4, "eight-push": 8, "four-staged": 4, "four-ll": 4}[mapping]
        mode = ("push" if "push" in mapping else "staged" if "staged" in mapping
                else "ll" if "ll" in mapping else "pull")
        summ = plan.schedule_summary(num_execs=execs, copy_mode=mode, verify=True)
        if mode not in ("staged", "ll"):
            assert summ["max_phases"] == 1  # no intra-slot hazards in reference plans
        assert sum(e["items"] for e in summ["execs"]) == summ["items"]


def test_write_groups_follow_id_order():
    # AR multi on flat {8}: slot 0 = one group per destination rank with
    # the init copy first and 7 reduces (SURVEY §7 hard part 1).
    plan, _, _ = harness.make_plan(7, 1, 8, 64, 0, 0, [8], 8, 1, 1, 1)
    summ = plan.schedule_summary(num_execs=8)
    ts = plan.transfer_dicts()
    groups = [it for it in summ["item_list"] if it["n_src"] == 8]
    assert len(groups) == 8
    for it in groups:
        ids = it["transfers"]
        assert ids == sorted(ids)
        assert not ts[ids[0]]["reduce"] and all(ts[i]["reduce"] for i in ids[1:])
        assert [ts[i]["src"] for i in ids] == list(range(8))  # ascending src
    # slot 1: 56 in-place copies, pulled by their destination
    copies = [it for it in summ["item_list"] if it["n_src"] == 1]
    assert len(copies) == 56 and all(it["exec"] == it["dst_rank"] for it in copies)


def test_push_mode_moves_copies_to_source():
    plan, _, _ = harness.make_plan(5, 0, 4, 100, 0, 0, [4], 4, 1, 1, 1)
    summ = plan.schedule_summary(num_execs=4, copy_mode="push")
    ts = plan.transfer_dicts()
    for it in summ["item_list"]:
        src = ts[it["transfers"][0]]["src"]
        assert it["exec"] == src


def test_virtual_ranks_arena_only_for_touching_ranks():
    # {2,4} g=4 stripe 4: staging buffers are declared for all ranks at full
    # length by the reference (factorize.cpp:85-86); the arena holds only
    # what each rank touches.
    plan, _, _ = harness.make_plan(7, 1, 8, 1 << 16, 0, 0, [2, 4], 4, 2, 4, 1)
    summ = plan.schedule_summary(num_execs=8, verify=False)
    declared = sum(length for name, length, inp, internal in plan.buffers if internal) * 4
    used = max(e["arena_bytes"] for e in summ["execs"])
    assert used < declared


def test_rejects_bad_mapping():
    plan, _, _ = harness.make_plan(7, 1, 8, 16, 0, 0, [8], 8, 1, 1, 1)
    with pytest.raises(H.HicclError) as e:
        plan.schedule_summary(num_execs=3)
    assert e.value.code == "InvalidConfig"


def test_push_reduce_chain_is_pure_push():
    # reduce over the chain 3 -> 2 -> 1 -> 0 (g = 1, ring 4, m = 4): the
    # reference initializes each accumulator with a copy and folds into it a
    # slot later; push schedules start the fold from the copy's source
    # (one item per hop and channel) and keep each accumulator in the arena
    # of the executor that reads it, so every hop is a remote store and
    # every load is local.
    plan, _, _ = harness.make_plan(3, 0, 4, 4096, 0, 0, [4], 1, 4, 1, 4)
    push = plan.schedule_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], copy_mode="push")
    pull = plan.schedule_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], copy_mode="pull")
    assert push["items"] < pull["items"]
    for it in push["item_list"]:
        assert not it["reads_dst"]
        if it["dst_buffer"].startswith("__acc"):
            assert it["dst_home"] == it["dst_rank"] - 1
        else:
            assert it["dst_home"] == it["dst_rank"]
    for it in pull["item_list"]:
        assert it["dst_home"] == it["exec"] or not it["dst_buffer"].startswith("__acc")


@pytest.mark.parametrize("kind,form", [(3, 0), (3, 1), (7, 1), (7, 2), (6, 1), (1, 0)])
def test_deferred_init_replays_reference(kind, form):
    # the fused schedules replay the reference's sequential fold order
    # (verify=1) on hierarchical, striped, ring and pipelined plans
    for hier, g, s, n, m in MACHINES:
        plan, _, _ = harness.make_plan(kind, form, 8, 37, 3 if kind < 4 else 0, 0, hier, g, n, s, m)
        for execs in (2, 4, 8):
            plan.schedule_summary(num_execs=execs, copy_mode="push", verify=True)


def test_push_reduce_multi_forwards_to_root():
    # reduce `multi` = reduce-scatter into __tmp, fence, gather to the root
    # (presets.cpp:145-161): push schedules store each fold straight into the
    # root's recvbuf (one item per executor, one step); pull keeps both steps
    plan, _, _ = harness.make_plan(3, 1, 4, 1024, 2)
    push = plan.schedule_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], copy_mode="push")
    assert push["items"] == 4
    for it in push["item_list"]:
        assert it["dst_rank"] == 2 and it["dst_buffer"] == "recvbuf" and it["step"] == 0
        assert len(it["transfers"]) == 5  # 4 folds + the forwarded gather copy
    pull = plan.schedule_summary(num_execs=4, rank_to_exec=[0, 1, 2, 3], copy_mode="pull")
    assert pull["items"] == 8
