"""BASELINE.json's configurations as parity cases on the GPUs available
(8 logical ranks spread over 4 or 2 B200s, or over two executors sharing
one), bit for bit against the oracle replaying the reference's plan.

C1 all-reduce 64 MiB/rank fp32, p=8, virtual {2,4}, tree and ring, s in {1,4},
   m in {1,4,16} (full size for one configuration, reduced for the grid)
C2 broadcast (single, multi) / scatter / gather on flat {8}
C3 all-reduce fp32/bf16 across sizes with pipelining (sizes up to 64 MiB)
C4 all-gather / reduce-scatter on the 3-level {2,2,2} (g=8, and g=2 with s=2)
C5 all-to-all on {8} and on {2,4} g=4 ring=2
"""
import pytest

import oracle
from tests import harness

pytestmark = pytest.mark.gpu
REF = oracle.Reference() if oracle.reference_available() else None


def devices():
    """4 or 2 GPUs when present, else two executors sharing the one GPU."""
    import torch
    n = torch.cuda.device_count()
    return harness.gpus(4 if n >= 4 else 2)


def run(kind, form, p, d, hier, g, s, n, m, dtype="f32", root=0, op=0, threads=1):
    plan, _, _ = harness.make_plan(kind, form, p, d, root, op, hier, g, n, s, m)
    flat = harness.oracle_plan(plan, kind, form, p, d, root, op, hier, g, n, s, m, REF)
    want = harness.run_oracle(flat, plan, dtype, 2024, threads=threads)
    got, _ = harness.run_device(plan, dtype, 2024, devices=devices())
    harness.assert_bitwise(got, want, f"{kind}/{form} {hier} g={g} s={s} n={n} m={m} {dtype}")


def test_c1_full_size():
    # 64 MiB per rank: p*d = 16,777,216 fp32
    run(7, 1, 8, 1 << 21, [2, 4], 4, 4, 2, 4, threads=8)


@pytest.mark.parametrize("s", [1, 4])
@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("m", [1, 4, 16])
def test_c1_grid(s, n, m):
    run(7, 1, 8, 65536 + 7, [2, 4], 4, s, n, m)


@pytest.mark.parametrize("kind,form", [(1, 0), (1, 1), (0, 0), (2, 0)])
@pytest.mark.parametrize("root", [0, 5])
def test_c2_rooted_flat8(kind, form, root):
    run(kind, form, 8, 1 << 20, [8], 8, 1, 1, 1, root=root)


def test_c2_broadcast_chain_ring8():
    # the pipelined chain over 8 "nodes" (g=1) that makes broadcast link-optimal
    run(1, 0, 8, 1 << 18, [2, 2, 2], 1, 1, 8, 8, root=3)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("d", [128, 65536, 1 << 21])
@pytest.mark.parametrize("m", [1, 8])
def test_c3_all_reduce_sizes(dtype, d, m):
    run(7, 1, 8, d, [8], 8, 1, 1, m, dtype=dtype)


@pytest.mark.parametrize("kind", [5, 6])
@pytest.mark.parametrize("g,s", [(8, 1), (2, 2)])
def test_c4_three_level(kind, g, s):
    run(kind, 0, 8, 1 << 18, [2, 2, 2], g, s, 1, 2)


@pytest.mark.parametrize("hier,g,n", [([8], 8, 1), ([2, 4], 4, 2)])
@pytest.mark.parametrize("m", [1, 4])
def test_c5_all_to_all(hier, g, n, m):
    run(4, 0, 8, 1 << 17, hier, g, 1, n, m)
