"""Plan parity: hiccl's factorizer + pipeliner against the reference's.

The executor reproduces the reference's fold order, so the plan — which
writer initializes each accumulator, canonical ids, stages, slots, deps,
staging-buffer names — must be identical to the reference's
(factorize.cpp:587-662, pipeline.cpp:76-132). The check is on the
serialized hiercoll-pipelined-v1 text, byte for byte.

Configurations where the reference ring lowering silently drops block
members (g=1 with ring blocks no hierarchy level groups) are
rejected by hiccl with InvalidConfig; for every such config the reference's
own plan must fail its own symbolic oracle.
"""
import itertools
import json
from pathlib import Path

import pytest

import oracle
from paper_2408_05962_b200 import hiccl as H

GOLDEN = Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")

FORMS = {0: [0], 1: [0, 1], 2: [0], 3: [0, 1], 4: [0], 5: [0, 1], 6: [0, 1], 7: [0, 1, 2]}


def mine(kind, form, p, count, root, op, hier, g, s, n, m):
    spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), root, count, H.ReduceOp(op))
    try:
        plan = H.lower(H.build(spec, p), H.Machine(list(hier), g), ring=n, stripe=s, pipeline=m)
    except H.HicclError as e:
        return e.status, str(e)
    return 0, plan.serialize()


def grid(ps=(4, 8, 12), counts=(1, 7), depths=(1, 3)):
    hiers = {4: [[4], [2, 2]], 6: [[6], [2, 3]], 8: [[8], [2, 4], [4, 2], [2, 2, 2]],
             12: [[12], [4, 3], [2, 2, 3], [3, 2, 2]]}
    for p in ps:
        for hier in hiers[p]:
            gs = {1, p}
            prod = 1
            for h in reversed(hier):
                prod *= h
                gs.add(prod)
            for g in sorted(gs):
                nodes = p // g
                for kind, fs in FORMS.items():
                    for form in fs:
                        for root in ([0, p - 1] if kind in (0, 1, 2, 3) else [0]):
                            for s in sorted({1, min(2, g), g}):
                                for n in sorted({1, nodes} | ({2} if nodes % 2 == 0 else set())):
                                    for m in depths:
                                        for count in counts:
                                            yield kind, form, p, count, root, 0, hier, g, s, n, m


@needs_ref
def test_plans_byte_identical_to_reference():
    ref = oracle.Reference()
    same = rejected = 0
    for cfg in grid():
        a = mine(*cfg)
        b = ref.preset_plan(*cfg[:7], cfg[7], cfg[8], cfg[9], cfg[10])
        if a[0] == 0:
            assert b[0] == 0, (cfg, b)
            assert a[1] == b[1], f"plan differs for {cfg}"
            same += 1
        elif a[0] == 9 and b[0] == 0 and "drop members" in a[1]:
            # hiccl refuses; the reference plan must be wrong by its own oracle
            kind, form, p, count, root, op = cfg[:6]
            rc, msg = ref.check_plan(b[1], kind, form, p, count, root, op)
            assert rc == 1, f"rejected config {cfg} but the reference plan passes: {msg}"
            rejected += 1
        else:
            assert a[0] == b[0], (cfg, a, b)
    assert same > 3000 and rejected > 0


@needs_ref
@pytest.mark.parametrize("op", [0, 1])
def test_reduction_ops_and_large_counts(op):
    ref = oracle.Reference()
    for cfg in [(7, 1, 8, 1 << 20, 0, op, [2, 4], 4, 4, 2, 16),
                (7, 0, 8, 12345, 0, op, [2, 2, 2], 2, 2, 4, 5),
                (6, 1, 8, 999, 0, op, [2, 2, 2], 8, 1, 1, 7),
                (3, 1, 12, 5001, 7, op, [3, 2, 2], 4, 4, 3, 2)]:
        a, b = mine(*cfg), ref.preset_plan(*cfg)
        assert a[0] == b[0] == 0 and a[1] == b[1], cfg


@needs_ref
def test_custom_program_lowering_matches_reference():
    """Non-preset compositions (mixed steps, in-place, overlapping roots)."""
    ref = oracle.Reference()
    p = 6
    prog = H.CollectiveProgram(p)
    prog.declare_buffer("a", 40, input=True).declare_buffer("b", 40).declare_buffer("c", 12)
    prog.add_reduction(H.BufferRef("a", 0, 10), H.BufferRef("b", 3, 10), [0, 2, 3, 5], 1)
    prog.add_multicast(H.BufferRef("a", 10, 7), H.BufferRef("b", 20, 7), 4, [0, 1, 2, 3, 4, 5])
    prog.add_fence()
    prog.add_multicast(H.BufferRef("b", 3, 10), H.BufferRef("c", 1, 10), 1, [5, 3])
    prog.add_reduction(H.BufferRef("b", 20, 7), H.BufferRef("b", 30, 7), [0, 1, 4], 2, H.ReduceOp.max)
    for hier, g, s, n, m in [([6], 6, 1, 1, 1), ([2, 3], 3, 3, 2, 4), ([3, 2], 2, 2, 3, 2),
                             ([3, 2], 1, 1, 6, 3)]:
        try:
            text = H.lower(prog, H.Machine(hier, g), ring=n, stripe=s, pipeline=m).serialize()
            rc_mine = 0
        except H.HicclError as e:
            rc_mine, text = e.status, str(e)
        rc, theirs = ref.lower_program(prog.serialize(), hier, g, s, n, m)
        if rc_mine == 0:
            assert rc == 0 and text == theirs, (hier, g, s, n, m)
            rc2, msg = ref.check_program_plan(prog.serialize(), text)
            assert rc2 == 0, msg
        else:
            assert rc_mine == 9 and rc == 0


def test_golden_plans():
    """Reference plans committed under tests/golden (made by
    tests/golden/make_golden.py from the reference library) — checked even
    where the reference cannot be built."""
    files = sorted(GOLDEN.glob("plan_*.json"))
    assert files, "golden fixtures missing"
    for f in files:
        meta = json.loads(f.with_suffix(".meta").read_text())
        rc, text = mine(*meta["config"])
        assert rc == 0, (f.name, text)
        assert text == f.read_text(), f.name


def test_misaligned_ring_rejected():
    # {8} g=1 ring=2: blocks of 4 ranks no level below the root groups.
    rc, msg = mine(7, 1, 8, 4, 0, 0, [8], 1, 1, 2, 1)
    assert rc == 9 and "drop members" in msg
    # all-to-all on the same machine has one member per block: nothing to drop
    assert mine(4, 0, 8, 4, 0, 0, [8], 1, 1, 2, 1)[0] == 0


def test_determinism():
    cfg = (7, 1, 8, 1000, 0, 0, [2, 4], 4, 4, 2, 4)
    assert mine(*cfg) == mine(*cfg)


def deep_grid():
    """SPEC.md:563's larger machines: p = 24 ({24}, {3,8}, {2,2,6}) and the
    4-level Frontier-like {2,2,4,2} (p = 32) and Aurora-like {2,2,6,2}
    (p = 48), g = the node size (the trailing factors), s in {1, g},
    ring in {1, node count}, m in {1, 4}."""
    for p, hier, g in [(24, [24], 24), (24, [3, 8], 8), (24, [2, 2, 6], 6),
                       (32, [2, 2, 4, 2], 8), (48, [2, 2, 6, 2], 12)]:
        nodes = p // g
        for kind, fs in FORMS.items():
            for form in fs:
                for s in sorted({1, g}):
                    for n in sorted({1, nodes}):
                        for m in (1, 4):
                            yield kind, form, p, 5, p - 1 if kind < 4 else 0, 0, hier, g, s, n, m


@needs_ref
def test_deep_hierarchies_byte_identical_to_reference():
    ref = oracle.Reference()
    same = 0
    for cfg in deep_grid():
        a = mine(*cfg)
        b = ref.preset_plan(*cfg[:7], cfg[7], cfg[8], cfg[9], cfg[10])
        assert a[0] == b[0], (cfg, a[1][:200], b[1][:200] if b[0] else b)
        if a[0] == 0:
            assert a[1] == b[1], f"plan differs for {cfg}"
            same += 1
    assert same > 300
