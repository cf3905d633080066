"""One process per GPU: IPC bootstrap of the executors.

The paper bootstraps with MPI; here any ``allgather(obj) ->
list`` works — torch.distributed.all_gather_object over gloo in bench.py
and the multi-process tests. No collective library is on the data path:
after ``connect()`` every peer buffer, arena and flag array is mapped
through CUDA IPC and the persistent kernels talk over NVLink directly.
"""
from __future__ import annotations

from typing import Callable, Sequence

from . import hiccl as H


class DistCommunicator:
    def __init__(self, plan: H.Plan, exec_index: int, num_execs: int, device: int,
                 dtype: str = "f32", rank_to_exec: Sequence[int] | None = None, **exec_kw):
        exec_kw.setdefault("copy_mode", "auto")  # push or tagged lines, by the cost model
        self.plan = plan
        self.exec_index = exec_index
        self.num_execs = num_execs
        self.device = device
        self.rank_to_exec = list(rank_to_exec) if rank_to_exec is not None else \
            H.split_ranks(plan.world_size, num_execs)
        self.executor = H.Executor(plan, device=device, exec_index=exec_index,
                                   num_execs=num_execs, rank_to_exec=self.rank_to_exec,
                                   dtype=dtype, **exec_kw)
        self._local: list[tuple[int, str, int, int]] = []
        self._imported: dict[bytes, int] = {}

    @property
    def local_ranks(self) -> list[int]:
        return [r for r, e in enumerate(self.rank_to_exec) if e == self.exec_index]

    def register(self, rank: int, name: str, ptr: int, nbytes: int) -> None:
        """Bind a buffer of a rank this process serves (device pointer on `device`)."""
        if self.rank_to_exec[rank] != self.exec_index:
            raise H.HicclError(2, f"RankOutOfRange: rank {rank} is served by executor "
                                  f"{self.rank_to_exec[rank]}, not {self.exec_index}")
        self.executor.bind_buffer(rank, name, ptr, nbytes)
        self._local.append((rank, name, ptr, nbytes))

    def enable_nvls(self, sizes: dict[str, int], allgather: Callable[[object], list]) -> dict:
        """Collective: put this process's rank buffers `name -> bytes` in one
        NVLS window (one rank per process) and bind unicast + multicast
        addresses for every rank. Returns name -> local device address."""
        if len(self.local_ranks) != 1 or self.plan.world_size != self.num_execs:
            raise H.HicclError(9, "InvalidConfig: NVLS needs one rank per process")
        rank = self.local_ranks[0]
        offs, total = H.window_layout(sizes)
        self.window_offsets = offs
        handle = self.window_handle = None
        if self.exec_index == 0:
            self.window = H.Window.open(self.device, self.num_execs, total, None)
            handle = self.window.export()
        handles = allgather(handle)
        if self.exec_index != 0:
            self.window = H.Window.open(self.device, self.num_execs, total, handles[0])
        allgather(None)  # every member added its device before anyone binds
        self.window.bind()
        uc, mc, _ = self.window.pointers(0)
        mems = allgather(self.window.export_memory())
        peers_uc = {}
        for e, h in enumerate(mems):
            if e != self.exec_index:
                peers_uc[e] = self.window.import_memory(h)
        allgather(None)
        self.window_bases = (uc, mc, peers_uc)
        return self._bind_window(offs, sizes)

    def share_nvls(self, owner: "DistCommunicator", offsets: dict[str, int],
                   sizes: dict[str, int]) -> dict:
        """Bind buffers `name -> bytes` at byte `offsets` inside the NVLS
        window `owner` created (owner.close() releases it; close this one
        first). Local, no exchange. Returns name -> local device address."""
        self.window_bases = owner.window_bases
        return self._bind_window(offsets, sizes)

    def _bind_window(self, offs: dict[str, int], sizes: dict[str, int]) -> dict:
        uc, mc, peers_uc = self.window_bases
        for name, off in offs.items():
            self.executor.bind_multicast(name, mc + off)
            for r in range(self.plan.world_size):
                e = self.rank_to_exec[r]
                base = uc if e == self.exec_index else peers_uc[e]
                self.executor.bind_buffer(r, name, base + off, sizes[name])
        return {name: uc + off for name, off in offs.items()}

    def _open(self, handle: bytes, offset: int) -> int:
        if handle not in self._imported:
            self._imported[handle] = H.ipc_import(handle, 0, self.device)
        return self._imported[handle] + offset

    def blob(self) -> dict:
        arena_ptr, _ = self.executor.local_arena()
        flags_ptr, _ = self.executor.local_flags()
        return {
            "exec": self.exec_index,
            "arena": H.ipc_export(arena_ptr),
            "flags": H.ipc_export(flags_ptr),
            "buffers": [(r, n, *H.ipc_export(p), nb) for r, n, p, nb in self._local],
        }

    def connect(self, allgather: Callable[[object], list]) -> None:
        blobs = allgather(self.blob())
        for b in blobs:
            e = b["exec"]
            if e == self.exec_index:
                continue
            self.executor.bind_peer_arena(e, self._open(*b["arena"]))
            self.executor.bind_peer_flags(e, self._open(*b["flags"]))
            for rank, name, handle, off, nbytes in b["buffers"]:
                self.executor.bind_buffer(rank, name, self._open(handle, off), nbytes)
        self.executor.commit()

    def start(self, stream: int = 0) -> None:
        self.executor.start(stream)

    def wait(self) -> None:
        self.executor.wait()

    def close(self) -> None:
        self.executor.close()
        if getattr(self, "window", None) is not None:
            self.window.close()
            self.window = None
        for base in self._imported.values():
            try:
                H._check(H.lib.hc_ipc_close(H.C.c_void_p(base)))
            except H.HicclError:
                pass
        self._imported.clear()
