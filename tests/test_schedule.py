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


# ---------------------------------------------------------------------------
# Hand-made and random plans: the push rewrites (deferred init, copy
# forwarding) and the write-group / phase rules must keep the sequential
# (slot, id) semantics of engine.cpp:285-330 for any plan the schedule
# accepts; verify=True replays both and raises on a difference.

def _plan_text(world, bufs, xfers, n=8):
    import json
    ts = [dict(id=i, stage=slot, level=1, stripe=0, channel=0, slot=slot, src=s, dst=d,
               src_buffer=sb, src_offset=so, dst_buffer=db, dst_offset=do, count=c,
               op="sum" if red else "copy", step=0, deps=[])
          for i, (slot, s, sb, so, d, db, do, c, red) in enumerate(xfers)]
    nst = max(x[0] for x in xfers) + 1
    return json.dumps({
        "format": "hiercoll-pipelined-v1", "world_size": world, "element_size": 4, "stripe": 1,
        "ring": 1, "num_stages": nst, "source_program_id": "0",
        "buffers": [dict(id=b, length=n, input=b.startswith("in"), internal=b[0].isupper())
                    for b in sorted(bufs)],
        "fences": [], "transfers": ts, "pipeline": 1, "slots": nst})


REGRESSIONS = [
    # deferred init moved a read of R onto the fold into D; the next
    # candidate (R += in3) did not see it and dropped R's init copy
    (2, [(0, 0, "in1", 0, 0, "R", 0, 8, False), (1, 0, "R", 0, 0, "D", 0, 8, False),
         (2, 0, "in2", 0, 0, "D", 0, 8, True), (3, 0, "in0", 0, 0, "R", 0, 8, True),
         (4, 0, "D", 0, 0, "out", 0, 8, False), (4, 0, "R", 0, 1, "out", 0, 8, False)]),
    (1, [(0, 0, "in1", 0, 0, "B", 0, 4, False), (0, 0, "in0", 0, 0, "A", 0, 4, False),
         (0, 0, "in1", 0, 0, "C", 0, 4, False), (1, 0, "in0", 0, 0, "B", 0, 4, False),
         (1, 0, "C", 0, 0, "out", 0, 4, False), (2, 0, "B", 0, 0, "out", 0, 4, False),
         (3, 0, "A", 0, 0, "out", 0, 4, False)]),
    # copy forwarding: A's new write to B's destination must be indexed
    (1, [(0, 0, "in0", 0, 0, "E", 0, 8, False), (0, 0, "in1", 0, 0, "D", 0, 8, False),
         (1, 0, "D", 0, 0, "E", 0, 8, False), (2, 0, "E", 0, 0, "out", 0, 8, False)]),
    # identity copy after a fold in the same slot
    (1, [(1, 0, "in0", 0, 0, "B", 2, 4, True), (1, 0, "B", 0, 0, "B", 0, 8, False),
         (2, 0, "B", 4, 0, "out", 4, 4, False)]),
    # deferred init must not fold from the copy's source when the fold
    # also reads the accumulator as a later source
    (1, [(0, 0, "in1", 0, 0, "A", 0, 1, False), (1, 0, "A", 0, 0, "A", 0, 1, True),
         (4, 0, "A", 0, 0, "out", 1, 4, True)]),
]


@pytest.mark.parametrize("case", range(len(REGRESSIONS)))
@pytest.mark.parametrize("mode", ["pull", "push", "staged", "ll"])
def test_schedule_regressions(case, mode):
    world, xs = REGRESSIONS[case]
    bufs = {b for x in xs for b in (x[2], x[5])}
    plan = H.Plan.deserialize(_plan_text(world, bufs, xs))
    for execs in {1, world}:
        plan.schedule_summary(num_execs=execs, copy_mode=mode, verify=True)


def test_schedule_random_plans():
    """Random plans with partial, overlapping and aliased ranges: every
    schedule built must replay the sequential execution exactly; plans it
    cannot express must be refused with an error, never run wrong."""
    import random
    rng = random.Random(20241019)
    n = 8
    checked = 0
    for _ in range(400):
        world = rng.choice([1, 2, 4])
        xs = []
        for slot in range(rng.randint(1, 5)):
            for _ in range(rng.randint(1, 4)):
                c = rng.choice([n, n // 2, 2, 1])
                so = rng.randrange(n - c + 1)
                do = rng.choice([so, rng.randrange(n - c + 1)])
                xs.append((slot, rng.randrange(world), rng.choice(["in0", "in1", "A", "B", "C"]), so,
                           rng.randrange(world), rng.choice(["A", "B", "C", "out"]), do, c,
                           rng.random() < 0.4))
        bufs = {"in0", "in1", "A", "B", "C", "out"}
        plan = H.Plan.deserialize(_plan_text(world, bufs, xs, n))
        for execs in (e for e in (1, 2, 4) if e <= world and world % e == 0):
            for mode in ("pull", "push", "staged", "ll"):
                try:
                    plan.schedule_summary(num_execs=execs, copy_mode=mode, verify=True)
                    checked += 1
                except H.HicclError as e:
                    msg = str(e)
                    assert not any(k in msg for k in ("replay differs", "no wait edge", "lost")), \
                        f"{mode} x{execs}: {msg}\n{xs}"
    assert checked > 1000


@pytest.mark.parametrize("cfg", [(3, 0, 4, 1 << 18, 0, 0, [4], 1, 4, 1, 1),
                                 (1, 0, 4, 1 << 18, 2, 0, [4], 1, 4, 1, 2),
                                 (7, 1, 8, 1 << 14, 0, 0, [2, 4], 4, 2, 4, 4),
                                 (6, 0, 8, 1 << 14, 0, 0, [2, 2, 2], 2, 1, 2, 2)])
@pytest.mark.parametrize("mode", ["push", "pull"])
def test_tile_sync_waits_cover_every_hazard(monkeypatch, cfg, mode):
    """HICCL_TILE_SYNC=1: consumer tiles wait for the producer tiles they
    conflict with (progress values step * T + ordinal + 1). verify_sync
    replays every conflicting tile pair against those waits (and the step
    waits), on 4 / 2 executors and on one."""
    monkeypatch.setenv("HICCL_TILE_SYNC", "1")
    plan, _, _ = harness.make_plan(*cfg)
    for ne in (4 if cfg[2] == 4 else 2, 1):
        plan.schedule_summary(num_execs=ne, copy_mode=mode, verify=True)


# The segment replay every executor runs on its schedule at create / commit
# (replay_schedule, schedule.cpp): exact at any byte count, and it catches
# a damaged schedule — a fold out of order, a dropped source, an item that
# misses an element.
DAMAGE = {1: "fold order", 2: "dropped source", 3: "missed element"}


@pytest.mark.parametrize("cfg", [(7, 1, 4, 1 << 10, [4], 4, 1, 1, 1),
                                 (7, 0, 4, 1000, [4], 4, 1, 1, 3),
                                 (7, 1, 8, 1 << 12, [2, 4], 4, 2, 4, 4),
                                 (3, 1, 8, 4097, [2, 2, 2], 2, 2, 2, 2),
                                 (5, 0, 4, 999, [2, 2], 2, 1, 2, 2)])
@pytest.mark.parametrize("mode", ["pull", "push", "staged", "ll"])
@pytest.mark.parametrize("damage", [1, 2, 3])
def test_replay_catches_damaged_schedules(cfg, mode, damage):
    kind, form, p, d, hier, g, ring, stripe, m = cfg
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, hier, g, ring, stripe, m)
    plan.schedule_summary(num_execs=p, copy_mode=mode, verify=2)  # intact: passes
    if damage in (1, 2) and kind not in (3, 6, 7):
        pytest.skip("no fold to damage in a copy-only collective")
    with pytest.raises(H.HicclError, match="replay differs"):
        plan.schedule_summary(num_execs=p, copy_mode=mode, verify=16 + damage)


def test_replay_at_full_size():
    """BASELINE C1 and a pipelined all-reduce at 1 GiB (+ a ragged tail)
    per rank: the replay works on segments, so it runs at these sizes."""
    for cfg in [(7, 1, 8, (1 << 28) + 12345, [2, 4], 4, 2, 4, 4),
                (7, 0, 4, (1 << 28) + 3, [4], 4, 1, 4, 32)]:
        kind, form, p, d, hier, g, ring, stripe, m = cfg
        plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, hier, g, ring, stripe, m)
        plan.schedule_summary(num_execs=p, copy_mode="push", verify=2)
