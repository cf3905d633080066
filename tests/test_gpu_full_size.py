"""BASELINE.json's configurations at their stated sizes (1 GiB per rank),
8 logical ranks on the GPUs available (two executors sharing one GPU on a
one-GPU box), bit for bit against the oracle replaying the reference's own
plan (presets.cpp:116-226 compositions, factorize.cpp:587 lowering).

C2 broadcast single / multi, scatter, gather on flat {8}, roots 0 and 5
C3 all-reduce multi f32 / bf16 on {8}, m in {1, 8}
C4 all-gather / reduce-scatter single on {2,2,2}, g = 8 and g = 2 with s = 2
C5 all-to-all at 8 MiB and 1 GiB per rank on {8} and {2,4} g = 4 ring 2

Inputs are generated on the device by the same counter hash the oracle
uses (hc_device_fill == oracle.fill), and results come back one
(buffer, rank) at a time, so host memory stays at the oracle's state plus
one buffer (<= 17 GiB at 1 GiB per rank).
"""
import os

import numpy as np
import pytest

import oracle
from tests import harness

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
REF = oracle.Reference() if oracle.reference_available() else None
GiB = 1 << 30
SEED = 4242


def devices():
    import torch
    n = torch.cuda.device_count()
    return harness.gpus(4 if n >= 4 else 2)


def run_full(kind, form, S, hier, g, s, n, m, dtype="f32", root=0):
    import torch
    from paper_2408_05962_b200 import hiccl as H
    p = 8
    esz = H.ELEMENT_SIZE[dtype]
    d = S // (p * esz)
    plan, _, _ = harness.make_plan(kind, form, p, d, root, 0, hier, g, n, s, m)
    flat = harness.oracle_plan(plan, kind, form, p, d, root, 0, hier, g, n, s, m, REF)
    what = f"{kind}/{form} {hier} g={g} s={s} n={n} m={m} {dtype} root={root} S={S}"

    # device side: fill in place, run, keep the tensors
    devs = devices()
    world = H.World(plan, devs, dtype)
    tensors = {}
    try:
        for name, length, inp, internal in plan.buffers:
            if internal:
                continue
            for r in range(p):
                dev = world.device_of(r)
                t = torch.empty(length * esz, dtype=torch.uint8, device=f"cuda:{dev}")
                H.device_fill(dev, t.data_ptr(), length, dtype,
                              SEED if inp else oracle.SENTINEL_SEED, r)
                world.bind(r, name, t.data_ptr(), t.numel())
                tensors[(name, r)] = t
        for dv in set(devs):
            torch.cuda.synchronize(dv)
        world.commit()
        world.run()
        for dv in set(devs):
            torch.cuda.synchronize(dv)
    finally:
        world.close()

    # oracle on the host, every core
    want = harness.run_oracle(flat, plan, dtype, SEED, threads=os.cpu_count() or 1)
    for (name, r), t in sorted(tensors.items()):
        got = t.cpu().numpy()
        exp = want[name][r].view(np.uint8)
        if not np.array_equal(got, exp):
            bad = np.nonzero(got != exp)[0]
            raise AssertionError(f"{what}: {name}@rank{r} differs in {bad.size} bytes, "
                                 f"first at byte {bad[0]}")
        del got
    tensors.clear()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind,form", [(1, 0), (1, 1), (0, 0), (2, 0)])
@pytest.mark.parametrize("root", [0, 5])
def test_c2_rooted_1gib(kind, form, root):
    run_full(kind, form, GiB, [8], 8, 1, 1, 1, root=root)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("m", [1, 8])
def test_c3_all_reduce_1gib(dtype, m):
    run_full(7, 1, GiB, [8], 8, 1, 1, m, dtype=dtype)


@pytest.mark.parametrize("kind", [5, 6])
@pytest.mark.parametrize("g,s", [(8, 1), (2, 2)])
def test_c4_three_level_1gib(kind, g, s):
    run_full(kind, 0, GiB, [2, 2, 2], g, s, 1, 1)


@pytest.mark.parametrize("S", [8 << 20, GiB])
@pytest.mark.parametrize("hier,g,n", [([8], 8, 1), ([2, 4], 4, 2)])
def test_c5_all_to_all(S, hier, g, n):
    run_full(4, 0, S, hier, g, 1, n, 1)
