"""Device executor vs the oracle, bit for bit.

All p logical ranks run on one B200 (one executor serving every rank, the
"virtual ranks" emulation of SURVEY §8(e)); multi-GPU variants live in
test_gpu_multi.py. The oracle replays the reference's own plan with the
numeric restatement of run_transfers (engine.cpp:285-330).
"""
import itertools

import pytest

import oracle
from tests import harness

pytestmark = pytest.mark.gpu

REF = oracle.Reference() if oracle.reference_available() else None

FORMS = {0: [0], 1: [0, 1], 2: [0], 3: [0, 1], 4: [0], 5: [0, 1], 6: [0, 1], 7: [0, 1, 2]}

# (hierarchy, g, stripe, ring) on p = 8: flat, the two virtual hierarchies
# of BASELINE.json, striping and ring chains.
MACHINES = [([8], 8, 1, 1), ([2, 4], 4, 1, 1), ([2, 4], 4, 4, 2), ([2, 2, 2], 8, 1, 1),
            ([2, 2, 2], 2, 2, 4), ([2, 2, 2], 1, 1, 8)]


def _check(kind, form, p, d, hier, g, stripe, ring, m, dtype, op=0, root=0, seed=1234, **kw):
    plan, spec, prog = harness.make_plan(kind, form, p, d, root, op, hier, g, ring, stripe, m)
    flat = harness.oracle_plan(plan, kind, form, p, d, root, op, hier, g, ring, stripe, m, REF)
    want = harness.run_oracle(flat, plan, dtype, seed)
    got, _ = harness.run_device(plan, dtype, seed, **kw)
    harness.assert_bitwise(got, want, f"kind={kind} form={form} {hier} g={g} s={stripe} "
                                      f"n={ring} m={m} {dtype}")


@pytest.mark.parametrize("kind,form", [(k, f) for k, fs in FORMS.items() for f in fs])
@pytest.mark.parametrize("machine", MACHINES, ids=lambda m: f"{m[0]}g{m[1]}s{m[2]}n{m[3]}")
def test_all_collectives_f32(kind, form, machine):
    hier, g, s, n = machine
    _check(kind, form, 8, 1000, hier, g, s, n, 3, "f32")


@pytest.mark.parametrize("dtype", ["bf16", "f16", "i32", "i64", "f64", "u8"])
@pytest.mark.parametrize("kind,form", [(7, 1), (7, 0), (6, 0), (3, 1), (5, 0)])
def test_dtypes(dtype, kind, form):
    _check(kind, form, 8, 777, [2, 4], 4, 4, 2, 2, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_max_op(dtype):
    _check(7, 1, 8, 513, [2, 2, 2], 8, 1, 1, 4, dtype, op=1)
    _check(3, 0, 8, 513, [8], 8, 1, 1, 1, dtype, op=1, root=5)


@pytest.mark.parametrize("d", [1, 3, 4, 5, 127, 4096, 65537])
def test_ragged_sizes(d):
    # balanced_split offsets are arbitrary element counts: head/tail peeling
    # and the misaligned scalar path must give identical results.
    _check(7, 1, 4, d, [4], 4, 1, 1, 3, "f32")
    _check(4, 0, 4, d, [2, 2], 2, 2, 2, 7, "bf16")


@pytest.mark.parametrize("root", [0, 3, 7])
def test_rooted_nonzero_root(root):
    for kind, form in [(0, 0), (1, 1), (2, 0), (3, 1)]:
        _check(kind, form, 8, 300, [2, 4], 4, 2, 2, 2, "f32", root=root)


def test_p1_local_copy():
    _check(7, 0, 1, 1 << 20, [1], 1, 1, 1, 1, "f32")


def test_repeated_starts_epochs():
    # flags are epoch-tagged: several start()/wait() rounds on one executor
    plan, spec, prog = harness.make_plan(7, 1, 8, 5000, 0, 0, [2, 4], 4, 2, 4, 4)
    flat = harness.oracle_plan(plan, 7, 1, 8, 5000, 0, 0, [2, 4], 4, 2, 4, 4, REF)
    want = harness.run_oracle(flat, plan, "f32", 1234)
    got, _ = harness.run_device(plan, "f32", 1234, repeat=5)
    harness.assert_bitwise(got, want, "repeat")


@pytest.mark.parametrize("ctas,threads", [(1, 64), (3, 128), (148, 512), (296, 256)])
def test_launch_shapes(ctas, threads):
    plan, spec, prog = harness.make_plan(7, 1, 8, 40000, 0, 0, [2, 4], 4, 2, 4, 3)
    flat = harness.oracle_plan(plan, 7, 1, 8, 40000, 0, 0, [2, 4], 4, 2, 4, 3, REF)
    want = harness.run_oracle(flat, plan, "f32", 99)
    got, _ = harness.run_device(plan, "f32", 99, ctas=ctas, threads=threads)
    harness.assert_bitwise(got, want, f"ctas={ctas} threads={threads}")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind,form,hier,g,stripe,ring,m", [
    (7, 1, [2, 4], 4, 4, 2, 4), (5, 0, [8], 8, 1, 1, 1), (1, 0, [2, 2, 2], 1, 1, 8, 3),
    (6, 1, [8], 8, 1, 1, 2), (3, 1, [2, 4], 4, 2, 1, 1)])
def test_unaligned_user_pointers(dtype, kind, form, hier, g, stripe, ring, m):
    """User buffers bound at pointers 0-3 elements past an allocation's
    start, different per rank and buffer: no item is 16-byte aligned or
    congruent across ranks for sure, so the TMA and staged paths must step
    aside and the vector / scalar bodies peel correctly."""
    esz = 4 if dtype == "f32" else 2
    plan, _, _ = harness.make_plan(kind, form, 8, 4099, 0, 0, hier, g, ring, stripe, m)
    flat = harness.oracle_plan(plan, kind, form, 8, 4099, 0, 0, hier, g, ring, stripe, m, REF)
    want = harness.run_oracle(flat, plan, dtype, 55)
    got, _ = harness.run_device(plan, dtype, 55,
                                misalign=lambda r, name: ((r + len(name)) % 4) * esz)
    harness.assert_bitwise(got, want, f"unaligned {kind}/{form} {hier} {dtype}")
