"""Multi-executor parity: 2-4 executors exchanging data, on 2-4 B200s over
NVLink when the box has them, else sharing one GPU (harness.gpus: each
executor its own stream and 1/n of the SMs; the protocol under test —
entry/exit barriers, system-scope step flags, peer loads/stores, staged
and tagged-line transfers, the IPC bootstrap — is the same).

Single process, one executor per device with peer access (World), and one
process per executor with the CUDA-IPC bootstrap (DistCommunicator). Ranks
map contiguously onto executors, so p = 8 on 2 or 4 executors also
exercises executors serving several logical ranks. Every result is
compared bit for bit with the oracle replaying the reference's plan.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from tests import harness

pytestmark = pytest.mark.gpu

REF = oracle.Reference() if oracle.reference_available() else None


def ngpu():
    import torch
    return torch.cuda.device_count()


TWO = lambda: harness.gpus(2)
FOUR = lambda: harness.gpus(4)


FORMS = [(k, f) for k, fs in {0: [0], 1: [0, 1], 2: [0], 3: [0, 1], 4: [0], 5: [0, 1],
                              6: [0, 1], 7: [0, 1, 2]}.items() for f in fs]


def _check(kind, form, p, d, hier, g, s, n, m, dtype, devices, op=0, root=0, **kw):
    plan, _, _ = harness.make_plan(kind, form, p, d, root, op, hier, g, n, s, m)
    flat = harness.oracle_plan(plan, kind, form, p, d, root, op, hier, g, n, s, m, REF)
    want = harness.run_oracle(flat, plan, dtype, 4321)
    got, stats = harness.run_device(plan, dtype, 4321, devices=devices, **kw)
    harness.assert_bitwise(got, want, f"{kind}/{form} p={p} {hier} on {devices} {kw}")
    return stats


@pytest.mark.parametrize("kind,form", FORMS)
@pytest.mark.parametrize("copy_mode", ["pull", "push", "staged", "ll"])
def test_two_gpus_flat(kind, form, copy_mode):
    _check(kind, form, 2, 5000, [2], 2, 1, 1, 2, "f32", TWO(), copy_mode=copy_mode)


@pytest.mark.parametrize("kind,form", FORMS)
@pytest.mark.parametrize("copy_mode", ["push", "staged", "ll"])
def test_p8_on_two_gpus_virtual_hierarchy(kind, form, copy_mode):
    stats = _check(kind, form, 8, 999, [2, 4], 4, 4, 2, 3, "f32", TWO(), copy_mode=copy_mode)
    assert all(s["num_items"] > 0 for s in stats) or kind in (0, 2)


@pytest.mark.parametrize("dtype", ["bf16", "i32"])
def test_p4_dtypes(dtype):
    for kind, form in [(7, 1), (5, 0), (6, 0), (4, 0)]:
        _check(kind, form, 4, 4097, [4], 4, 1, 1, 4, dtype, FOUR())


@pytest.mark.parametrize("dtype", ["bf16", "f16", "i32", "u8", "i64", "f64"])
def test_ll_dtypes_ragged(dtype):
    # odd counts: partial tagged lines at every range end; repeat=3 runs
    # both arena copies (launch parity) and reuses the first one
    for kind, form in [(7, 1), (5, 0), (6, 0), (4, 0), (3, 1), (1, 1)]:
        _check(kind, form, 2, 1001, [2], 2, 1, 1, 3, dtype, TWO(), copy_mode="ll", repeat=3)


def test_ll_four_executors():
    for kind, form in FORMS:
        _check(kind, form, 4, 2049, [4], 4, 1, 1, 2, "f32", FOUR(), copy_mode="ll", repeat=2)
    _check(7, 1, 4, 1 << 18, [4], 4, 1, 1, 1, "bf16", FOUR(), copy_mode="ll", repeat=2)


def test_auto_copy_mode_follows_the_model():
    # small all-reduce -> tagged lines; 64 MiB per rank -> push; bit-exact both ways
    small = _check(7, 0, 2, 256, [2], 2, 1, 1, 1, "f32", TWO(), copy_mode="auto")
    assert all(st["copy_mode"] == 3 for st in small)
    big = _check(7, 1, 2, 1 << 23, [2], 2, 1, 1, 1, "f32", TWO(), copy_mode="auto")
    assert all(st["copy_mode"] == 1 for st in big)


def test_p8_on_four_executors_222():
    for kind, form in FORMS:
        _check(kind, form, 8, 777, [2, 2, 2], 2, 2, 4, 2, "f32", FOUR())


def test_large_all_reduce_two_executors():
    _check(7, 1, 2, 1 << 22, [2], 2, 1, 1, 1, "f32", TWO())
    _check(5, 0, 2, 1 << 22, [2], 2, 1, 1, 1, "bf16", TWO(), copy_mode="push")


# ---- one process per GPU, CUDA IPC bootstrap -------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _mp_worker(rank, world, port, kind, form, p, d, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_05962_b200 import hiccl as H
        from paper_2408_05962_b200.dist import DistCommunicator
        dev = rank % torch.cuda.device_count()  # one GPU: processes share it (time-sliced)
        torch.cuda.set_device(dev)
        plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 2)
        comm = DistCommunicator(plan, rank, world, device=dev, dtype="f32", timeout_s=60)
        init = harness.initial_state(plan, "f32", 777)
        keep = {}
        for r in comm.local_ranks:
            for name in init:
                t = torch.from_numpy(init[name][r].view(np.uint8).copy()).to(f"cuda:{dev}")
                keep[(name, r)] = t
                comm.register(r, name, t.data_ptr(), t.numel())

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        comm.connect(allgather)
        for _ in range(3):
            comm.start()
            comm.wait()
        torch.cuda.synchronize()
        dist.barrier()
        res = {k: v.cpu().numpy() for k, v in keep.items()}
        comm.close()
        q.put((rank, res))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,form,p", [(7, 1, 2), (5, 0, 2), (4, 0, 2), (7, 1, 4), (6, 0, 4)])
def test_one_process_per_gpu(kind, form, p):
    import torch.multiprocessing as mp
    world = 2  # processes; on a one-GPU box both share cuda:0
    d = 3001
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, kind, form, p, d, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(world):
        rank, res = q.get(timeout=180)
        assert not isinstance(res, str), res
        got.update(res)
    for pr in procs:
        pr.join(timeout=60)
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 2)
    flat = harness.oracle_plan(plan, kind, form, p, d, 0, 0, [p], p, 1, 1, 2, REF)
    want = harness.run_oracle(flat, plan, "f32", 777)
    for name, per_rank in want.items():
        for r in range(p):
            assert got[(name, r)].tobytes() == per_rank[r].view(np.uint8).tobytes(), (name, r)


@pytest.mark.parametrize("kind,form,p,copy_mode", [(7, 1, 2, "push"), (7, 1, 4, "pull"),
                                                   (4, 0, 4, "push"), (6, 1, 2, "push"),
                                                   (7, 1, 4, "staged"), (3, 1, 2, "staged"),
                                                   (7, 1, 2, "ll"), (7, 1, 4, "ll"),
                                                   (0, 0, 2, "ll"), (1, 0, 4, "ll")])
def test_back_to_back_epochs_with_changing_inputs(kind, form, p, copy_mode):
    """Epochs launched without host synchronization; between epochs every
    rank's inputs are rewritten on its stream and every epoch's output is
    snapshotted. Each snapshot must equal the oracle for that epoch's
    inputs: a missing cross-epoch ordering (a peer still reading my inputs
    or writing my outputs from the previous epoch) would corrupt one."""
    import torch
    from paper_2408_05962_b200 import hiccl as H
    d, epochs = 4099, (9 if copy_mode == "ll" else 6)
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 3)
    devices = TWO()
    world = H.World(plan, devices, "f32", copy_mode=copy_mode)
    esz = 4
    bufs, snaps = {}, {}
    try:
        for name, length, inp, internal in plan.buffers:
            if internal:
                continue
            for r in range(p):
                dev = world.device_of(r)
                t = torch.zeros(length * esz, dtype=torch.uint8, device=f"cuda:{dev}")
                bufs[(name, r)] = (t, length, inp)
                world.bind(r, name, t.data_ptr(), t.numel())
        world.commit()
        # one stream per executor (executors may share a GPU): a rank's
        # fills and snapshots are ordered with its executor only; ordering
        # against the other executors is the kernel's entry/exit barrier
        streams = [torch.cuda.Stream(dv) for dv in devices]
        for e in range(epochs):
            for (name, r), (t, length, inp) in bufs.items():
                if inp:
                    x = world.rank_to_exec[r]
                    H.device_fill(devices[x], t.data_ptr(), length, "f32", 1000 + e, r,
                                  stream=streams[x].cuda_stream)
            for i, ex in enumerate(world.execs):
                ex.start(streams[i].cuda_stream)
            for (name, r), (t, length, inp) in bufs.items():
                if not inp:
                    x = world.rank_to_exec[r]
                    with torch.cuda.stream(streams[x]):
                        snaps[(e, name, r)] = t.clone()
        world.wait()
        for dv in set(devices):
            torch.cuda.synchronize(dv)
        flat = harness.oracle_plan(plan, kind, form, p, d, 0, 0, [p], p, 1, 1, 3, REF)
        for e in range(epochs):
            st = {}
            for name, length, inp, internal in plan.buffers:
                if internal:
                    continue
                st[name] = [oracle.fill(length, "f32", 1000 + e, r) if inp else
                            (np.zeros(length, np.float32) if e == 0 else want_prev[name][r].copy())
                            for r in range(p)]
            oracle.execute(flat, "f32", st)
            for (ee, name, r), snap in snaps.items():
                if ee == e:
                    assert snap.cpu().numpy().tobytes() == st[name][r].tobytes(), (e, name, r)
            want_prev = st
    finally:
        world.close()


# ---- watchdog ---------------------------------------------------------------

@pytest.mark.parametrize("copy_mode", ["push", "pull"])
def test_watchdog_timeout_poisons_the_executor(copy_mode):
    """A peer that never starts: executor 0's entry barrier waits for a
    flag nobody publishes. The wait must come back as HC_TIMEOUT (15) after
    the watchdog, not hang the GPU, and the executor must refuse further
    launches (its flag epochs are no longer in step with its peers)."""
    import time
    import torch
    from paper_2408_05962_b200 import hiccl as H
    plan, _, _ = harness.make_plan(7, 1, 2, 4096, 0, 0, [2], 2, 1, 1, 1)
    devs = TWO()
    world = H.World(plan, devs, "f32", copy_mode=copy_mode, timeout_s=1.0)
    keep = []
    try:
        for name, length, inp, internal in plan.buffers:
            if internal:
                continue
            for r in range(2):
                t = torch.zeros(length * 4, dtype=torch.uint8, device=f"cuda:{world.device_of(r)}")
                keep.append(t)
                world.bind(r, name, t.data_ptr(), t.numel())
        world.commit()
        t0 = time.time()
        world.execs[0].start()  # executor 1 is never launched
        with pytest.raises(H.HicclError) as e:
            world.execs[0].wait()
        assert e.value.status == 15 and e.value.code == "Timeout", e.value
        assert time.time() - t0 < 30
        with pytest.raises(H.HicclError) as e2:
            world.execs[0].start()
        assert e2.value.status == 15
        # the device is still usable
        x = torch.ones(1024, device=f"cuda:{devs[0]}")
        assert float(x.sum()) == 1024.0
    finally:
        world.close()


# ---- re-commit -----------------------------------------------------------------

@pytest.mark.parametrize("copy_mode", ["push", "ll"])
def test_recommit_after_launches_and_graph_replays(copy_mode):
    """commit() again after launches — plain and CUDA-graph-replayed ones,
    which the host never counts — and keep going with new inputs: the
    epoch lives on the device and the exit counter is per launch, so the
    flags of the re-committed executors stay in step (a stale flag would
    let a consumer read a previous epoch's data). Every epoch is checked
    against the oracle."""
    import torch
    from paper_2408_05962_b200 import hiccl as H
    p, d = 2, 2053
    plan, _, _ = harness.make_plan(7, 1, p, d, 0, 0, [p], p, 1, 1, 2)
    devices = TWO()
    flat = harness.oracle_plan(plan, 7, 1, p, d, 0, 0, [p], p, 1, 1, 2, REF)
    world = H.World(plan, devices, "f32", copy_mode=copy_mode)
    bufs = {}
    try:
        for name, length, inp, internal in plan.buffers:
            if internal:
                continue
            for r in range(p):
                t = torch.zeros(length * 4, dtype=torch.uint8, device=f"cuda:{world.device_of(r)}")
                bufs[(name, r)] = (t, length, inp)
                world.bind(r, name, t.data_ptr(), t.numel())
        streams = [torch.cuda.Stream(dv) for dv in devices]

        def epoch(seed, graphs=None):
            for (name, r), (t, length, inp) in bufs.items():
                if inp:
                    H.device_fill(world.device_of(r), t.data_ptr(), length, "f32", seed, r)
            for dv in set(devices):
                torch.cuda.synchronize(dv)
            if graphs:  # each executor's graph on its own stream (they run concurrently)
                for i, g in enumerate(graphs):
                    with torch.cuda.device(devices[i]), torch.cuda.stream(streams[i]):
                        g.replay()
            else:
                for i, ex in enumerate(world.execs):
                    ex.start(streams[i].cuda_stream)
            for dv in set(devices):
                torch.cuda.synchronize(dv)
            world.wait()
            st = {name: [oracle.fill(length, "f32", seed, r) if inp else np.zeros(length, np.float32)
                         for r in range(p)]
                  for name, length, inp, internal in plan.buffers if not internal}
            oracle.execute(flat, "f32", st)
            for (name, r), (t, length, inp) in bufs.items():
                if not inp:
                    assert t.cpu().numpy().tobytes() == st[name][r].tobytes(), (seed, name, r)

        world.commit()
        for e in range(3):
            epoch(100 + e)
        # capture one launch per executor, replay it (host never sees these)
        graphs = []
        for i, ex in enumerate(world.execs):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.device(devices[i]), torch.cuda.graph(g, stream=streams[i]):
                ex.start(streams[i].cuda_stream)
            graphs.append(g)
        for e in range(3):
            epoch(200 + e, graphs)
        world.commit()  # re-commit after plain and replayed launches
        for e in range(3):
            epoch(300 + e)
    finally:
        world.close()


# ---- checked mode (runtime dependency check) --------------------------------

@pytest.fixture
def checked_env(monkeypatch):
    monkeypatch.setenv("HICCL_CHECK_DEPS", "1")
    return monkeypatch


@pytest.mark.parametrize("kind,form,p,copy_mode,m", [(7, 1, 2, "pull", 1), (7, 1, 4, "push", 3),
                                                     (3, 1, 2, "staged", 2), (5, 1, 4, "pull", 2),
                                                     (7, 1, 2, "ll", 2), (4, 0, 4, "push", 1)])
def test_checked_mode_passes_on_correct_schedules(checked_env, kind, form, p, copy_mode, m):
    """HICCL_CHECK_DEPS=1: before each step every CTA re-reads the flag of
    every producer tile its tiles conflict with (engine.cpp:302-306's "deps
    done" check, at tile grain, on the device). Correct schedules pass and
    stay bit-exact."""
    _check(kind, form, p, 3001, [p], p, 1, 1, m, "f32", harness.gpus(p), copy_mode=copy_mode)


def test_checked_mode_catches_a_dropped_wait(checked_env):
    """Negative test (SPEC.md:392's corrupted dependency, on the device):
    every wait dropped and executor 1 slowed by 2 ms per step, so executor
    0 reaches the all-gather step (which pulls executor 1's reduced chunk)
    before executor 1 finished its reduce-scatter step. The launch must
    fail with DependencyViolation, not return wrong data."""
    from paper_2408_05962_b200 import hiccl as H
    checked_env.setenv("HICCL_TEST_DROP_WAITS", "1")
    checked_env.setenv("HICCL_TEST_DELAY_EXEC", "1")
    plan, _, _ = harness.make_plan(7, 1, 2, 4096, 0, 0, [2], 2, 1, 1, 1)
    with pytest.raises(H.HicclError) as e:
        harness.run_device(plan, "f32", 3, devices=TWO(), copy_mode="pull", timeout_s=3.0)
    assert e.value.code == "DependencyViolation", e.value
    assert "before CTA" in str(e.value)


# ---- tile-granular progress (HICCL_TILE_SYNC) ----------------------------------

@pytest.mark.parametrize("kind,form,p,hier,g,ring,m,mode", [
    (3, 0, 4, [4], 1, 4, 1, "push"),     # reduce chain, followed tile by tile
    (1, 0, 4, [4], 1, 4, 2, "pull"),     # broadcast chain, pipelined
    (7, 1, 4, [4], 4, 1, 3, "push"),     # all-reduce, pipelined
    (7, 1, 8, [2, 4], 4, 2, 2, "push"),  # C1-shaped, 8 ranks on the executors
])
def test_tile_sync_bit_exact(monkeypatch, kind, form, p, hier, g, ring, m, mode):
    """The tile-sync kernel variant: consumer tiles wait for exactly the
    producer tiles they conflict with, producers publish per tile."""
    monkeypatch.setenv("HICCL_TILE_SYNC", "1")
    _check(kind, form, p, 40961, hier, g, 1, ring, m, "f32", harness.gpus(min(p, 4)),
           copy_mode=mode)
