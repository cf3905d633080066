"""Edge cases at the limits: element counts past 2^31 and 2^32 (64-bit
indexing end to end), single-element and ragged buffers, and the
misaligned (scalar) path at scale. Results are checked on the device
against the collective's definition (copies / wrapping u8 sums are exact
under any order, so these are bit-exact checks)."""
import numpy as np
import pytest

from paper_2408_05962_b200 import hiccl as H
from tests import harness

pytestmark = pytest.mark.gpu


def _run(plan, dtype, fill_seed=9):
    import torch
    esz = H.ELEMENT_SIZE[dtype]
    world = H.World(plan, [0], dtype)
    bufs = {}
    try:
        for name, length, inp, internal in plan.buffers:
            if internal:
                continue
            for r in range(plan.world_size):
                t = torch.zeros(length * esz, dtype=torch.uint8, device="cuda:0")
                if inp:
                    H.device_fill(0, t.data_ptr(), length, dtype, fill_seed, r)
                bufs[(name, r)] = t
                world.bind(r, name, t.data_ptr(), t.numel())
        world.commit()
        world.run()
        torch.cuda.synchronize()
        return bufs
    finally:
        world.close()


def test_copy_past_2_pow_32_elements():
    import torch
    n = (1 << 32) + 4099  # u8 elements: > 2^32, ragged tail
    plan, _, _ = harness.make_plan(7, 0, 1, n, 0, 0, [1], 1, 1, 1, 1)
    bufs = _run(plan, "u8")
    assert torch.equal(bufs[("recvbuf", 0)], bufs[("sendbuf", 0)])


def test_reduce_past_2_pow_31_elements():
    import torch
    d = (1 << 31) + 17  # per-rank chunk; p*d > 2^32 u8 elements
    plan, _, _ = harness.make_plan(7, 1, 2, d, 0, 0, [2], 2, 1, 1, 1)
    bufs = _run(plan, "u8")
    want = bufs[("sendbuf", 0)] + bufs[("sendbuf", 1)]  # uint8 wraps
    assert torch.equal(bufs[("recvbuf", 0)], want)
    assert torch.equal(bufs[("recvbuf", 1)], want)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_tiny_counts_all_collectives(d):
    import oracle
    for kind, form in [(0, 0), (1, 1), (2, 0), (3, 1), (4, 0), (5, 1), (6, 1), (7, 2)]:
        plan, _, _ = harness.make_plan(kind, form, 4, d, 1 if kind < 4 else 0, 0, [2, 2], 2, 2, 2, 3)
        flat = oracle.FlatPlan.from_dicts(4, plan.buffers, plan.transfer_dicts())
        want = harness.run_oracle(flat, plan, "f32", 3)
        got, _ = harness.run_device(plan, "f32", 3)
        harness.assert_bitwise(got, want, f"tiny {kind}/{form} d={d}")


def test_misaligned_scalar_path_large():
    # offsets that are not congruent mod 16 between source and destination
    # (a custom composition), 40 MiB, bf16: the element-wise path
    import oracle
    p, n = 2, 20_000_003
    prog = H.CollectiveProgram(p)
    prog.declare_buffer("a", n + 8, input=True).declare_buffer("b", n + 8)
    prog.add_multicast(H.BufferRef("a", 1, n), H.BufferRef("b", 6, n), 0, [0, 1])
    prog.add_fence()
    prog.add_reduction(H.BufferRef("b", 6, n), H.BufferRef("b", 6, n), [0, 1], 1)
    plan = H.lower(prog, H.Machine([2], 2), pipeline=3)
    flat = oracle.FlatPlan.from_dicts(p, plan.buffers, plan.transfer_dicts())
    want = harness.run_oracle(flat, plan, "bf16", 8)
    got, _ = harness.run_device(plan, "bf16", 8)
    harness.assert_bitwise(got, want, "misaligned bf16")
