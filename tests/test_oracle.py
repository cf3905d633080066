"""Pinning the oracle before trusting it.

* the shared input generator against an independent pure-Python splitmix64
  and the committed known-answer vectors (tests/golden/fill_*.npy);
* the numeric restatement of run_transfers (oracle/numeric_exec.c) on the
  REFERENCE's own plans against independently computed collective results:
  exact for integer sums and max (any fold order gives the same answer),
  within 1e-6 of the sum of magnitudes for fp32;
* the reference's symbolic executor + ground truth (engine.cpp:285-347,
  presets.cpp:231-298) on hiccl's plans: dataflow identical (PASS);
* the negative test of SPEC.md:392: a plan with a transfer removed is caught.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2408_05962_b200 import hiccl as H
from tests import harness

GOLDEN = Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")

M64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def test_generator_known_answers():
    seed, rank, base = 1234, 3, 1000
    hs = [splitmix64(seed ^ (rank << 40) ^ (base + i)) for i in range(64)]
    f32 = np.array([((h >> 40) * 2.0 ** -24) * 2 - 1 for h in hs], dtype=np.float32)
    assert (oracle.fill(64, "f32", seed, rank, base) == f32).all()
    i32 = np.array([(h >> 33) & 0xFFFF for h in hs], dtype=np.int32)
    assert (oracle.fill(64, "i32", seed, rank, base) == i32).all()
    u8 = np.array([h >> 56 for h in hs], dtype=np.uint8)
    assert (oracle.fill(64, "u8", seed, rank, base) == u8).all()
    for dt in ("f32", "bf16", "f16", "i32", "i64", "f64", "u8"):
        want = np.load(GOLDEN / f"fill_{dt}.npy")
        assert oracle.fill(64, dt, seed, rank, base).tobytes() == want.tobytes(), dt


def test_bf16_rounding_is_rne():
    f = oracle.fill(4096, "f32", 7, 0)
    b = oracle.fill(4096, "bf16", 7, 0)
    u = f.view(np.uint32).astype(np.uint64)
    rne = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert (b == rne).all()


CASES = [(k, f) for k, fs in {0: [0], 1: [0, 1], 2: [0], 3: [0, 1], 4: [0], 5: [0, 1],
                              6: [0, 1], 7: [0, 1, 2]}.items() for f in fs]
MACHINES = [([8], 8, 1, 1, 1), ([2, 4], 4, 4, 2, 3), ([2, 2, 2], 2, 2, 4, 2),
            ([2, 2, 2], 8, 1, 1, 5), ([2, 2, 2], 1, 1, 8, 4)]


@pytest.mark.parametrize("kind,form", CASES)
@pytest.mark.parametrize("dtype,op", [("i32", 0), ("i64", 0), ("u8", 0), ("i32", 1), ("f32", 1)])
def test_numeric_oracle_exact_on_reference_plans(kind, form, dtype, op):
    ref = oracle.Reference() if oracle.reference_available() else None
    p, d = 8, 33
    for hier, g, s, n, m in MACHINES:
        root = 5 if kind in (0, 1, 2, 3) else 0
        plan, _, _ = harness.make_plan(kind, form, p, d, root, op, hier, g, n, s, m)
        flat = harness.oracle_plan(plan, kind, form, p, d, root, op, hier, g, n, s, m, ref)
        st = harness.initial_state(plan, dtype, 99)
        want = oracle.ground_truth(kind, p, d, root, op, dtype, st["sendbuf"], st["recvbuf"])
        oracle.execute(flat, dtype, st, track_defined=True)
        for r in range(p):
            assert st["recvbuf"][r].tobytes() == want[r].tobytes(), (kind, form, hier, r)


@pytest.mark.parametrize("kind,form", [(7, 0), (7, 1), (7, 2), (6, 0), (6, 1), (3, 0), (3, 1)])
def test_numeric_oracle_fp32_sum_within_tolerance(kind, form):
    p, d = 8, 257
    for hier, g, s, n, m in MACHINES:
        plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, hier, g, n, s, m)
        flat = oracle.FlatPlan.from_dicts(p, plan.buffers, plan.transfer_dicts())
        st = harness.initial_state(plan, "f32", 1234)
        sends = [x.astype(np.float64) for x in st["sendbuf"]]
        exact = np.sum(sends, axis=0)
        mag = np.sum(np.abs(sends), axis=0)
        oracle.execute(flat, "f32", st)
        owners = range(p) if kind == 7 else ([0] if kind == 3 else range(p))
        for r in owners:
            sl = slice(r * d, (r + 1) * d) if kind == 6 else slice(0, p * d)
            err = np.abs(st["recvbuf"][r][sl].astype(np.float64) - exact[sl]) / mag[sl]
            assert err.max() <= 1e-6


@needs_ref
@pytest.mark.parametrize("kind,form", CASES)
def test_reference_symbolic_oracle_passes_hiccl_plans(kind, form):
    """execute_plan(hiccl plan) == reference_semantics, exact symbolic
    equality (SPEC.md:563 grid, reduced)."""
    ref = oracle.Reference()
    for p, machines in [(8, MACHINES), (4, [([4], 4, 1, 1, 1), ([2, 2], 2, 2, 2, 3)]),
                        (12, [([3, 2, 2], 4, 4, 3, 2), ([12], 12, 1, 1, 4)])]:
        for hier, g, s, n, m in machines:
            for op in (0, 1):
                root = p - 1 if kind in (0, 1, 2, 3) else 0
                plan, _, _ = harness.make_plan(kind, form, p, 5, root, op, hier, g, n, s, m)
                rc, msg = ref.check_plan(plan.serialize(), kind, form, p, 5, root, op)
                assert rc == 0, (kind, form, p, hier, g, s, n, m, msg)


def test_dropped_transfer_is_detected():
    """SPEC.md:392 negative test: remove one transfer from a plan."""
    p, d = 8, 16
    plan, _, _ = harness.make_plan(7, 1, p, d, 0, 0, [2, 4], 4, 1, 4, 2)
    ts = plan.transfer_dicts()
    st0 = harness.initial_state(plan, "i32", 5)
    want = oracle.ground_truth(7, p, d, 0, 0, "i32", st0["sendbuf"], st0["recvbuf"])
    # drop one transfer of the first step
    victim = next(t for t in ts if t["step"] == 0 and t["reduce"])
    flat = oracle.FlatPlan.from_dicts(p, plan.buffers, [t for t in ts if t is not victim])
    st = harness.initial_state(plan, "i32", 5)
    try:
        oracle.execute(flat, "i32", st, track_defined=True)
    except RuntimeError as e:
        assert "UninitializedRead" in str(e)
        return
    assert any(st["recvbuf"][r].tobytes() != want[r].tobytes() for r in range(p))
