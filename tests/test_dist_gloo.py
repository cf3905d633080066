"""The N > 1 host path on CPU: two processes over gloo (127.0.0.1).

* every process lowers the same composition to the byte-identical plan and
  the same executor schedule (the paper's "every rank registers the same
  program");
* the IPC bootstrap of DistCommunicator binds exactly the peer arenas,
  flag words and user buffers the other process exported (CUDA IPC and the
  executor are replaced by recording fakes — no device on this host).
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeExecutor:
    def __init__(self, plan, device=0, exec_index=0, num_execs=1, rank_to_exec=None, dtype="f32",
                 **kw):
        self.exec_index = exec_index
        self.calls = []
        self._h = True

    def local_arena(self):
        return 0x1000_0000 + self.exec_index, 4096

    def local_flags(self):
        return 0x2000_0000 + self.exec_index, 512

    def bind_buffer(self, rank, name, ptr, nbytes):
        self.calls.append(("buffer", rank, name, ptr, nbytes))

    def bind_peer_arena(self, peer, ptr):
        self.calls.append(("arena", peer, ptr))

    def bind_peer_flags(self, peer, ptr):
        self.calls.append(("flags", peer, ptr))

    def commit(self):
        self.calls.append(("commit",))

    def close(self):
        pass


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_05962_b200 import dist as D
        from paper_2408_05962_b200 import hiccl as H

        prog = H.build(H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, 1000),
                       world * 2)
        plan = H.lower(prog, H.Machine([world, 2], 2), ring=world, stripe=2, pipeline=4)
        text = plan.serialize()
        summ = plan.schedule_summary(num_execs=world)
        texts = [None] * world
        dist.all_gather_object(texts, (text, summ["items"], summ["steps"]))

        # fake IPC: the handle carries the pointer; import adds a per-process base
        H.Executor = FakeExecutor
        D.H.Executor = FakeExecutor
        D.H.ipc_export = lambda ptr: (ptr.to_bytes(8, "little") * 8, 16)
        D.H.ipc_import = lambda h, off, dev: int.from_bytes(h[:8], "little") + 0x7000_0000 + off
        comm = D.DistCommunicator(plan, rank, world, device=rank)
        for r in comm.local_ranks:
            comm.register(r, "sendbuf", 0x3000_0000 + 0x100 * r, 8000)
            comm.register(r, "recvbuf", 0x4000_0000 + 0x100 * r, 8000)

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        comm.connect(allgather)
        q.put((rank, texts, comm.local_ranks, comm.executor.calls))
    finally:
        dist.destroy_process_group()


def test_two_process_bootstrap():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, texts, local, calls = q.get(timeout=120)
        results[rank] = (texts, local, calls)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    texts0 = results[0][0]
    assert all(t == texts0[0] for t in texts0)  # identical plans and schedules on both ranks
    for rank, (texts, local, calls) in results.items():
        peer = 1 - rank
        assert local == [2 * rank, 2 * rank + 1]
        assert ("arena", peer, 0x1000_0000 + peer + 0x7000_0000 + 16) in calls
        assert ("flags", peer, 0x2000_0000 + peer + 0x7000_0000 + 16) in calls
        bufs = sorted(c[1:] for c in calls if c[0] == "buffer")
        want = []
        for r in range(4):
            if r in local:
                want += [(r, "recvbuf", 0x4000_0000 + 0x100 * r, 8000),
                         (r, "sendbuf", 0x3000_0000 + 0x100 * r, 8000)]
            else:
                want += [(r, "recvbuf", 0x4000_0000 + 0x100 * r + 0x7000_0000 + 16, 8000),
                         (r, "sendbuf", 0x3000_0000 + 0x100 * r + 0x7000_0000 + 16, 8000)]
        assert bufs == sorted(want)
        assert calls[-1] == ("commit",)
