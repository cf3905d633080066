"""Python face of the C ABI (include/hiccl.h).

Mirrors the reference's public C++ API so tests and drivers read like the
reference's own code (proj/include/hiercoll/*.hpp):

    prog = CollectiveProgram(p)                       # composition.hpp:66
    prog.declare_buffer("sendbuf", n, input=True)
    prog.add_multicast(BufferRef(...), BufferRef(...), root, leaves)
    prog.add_reduction(send, recv, leaves, root, ReduceOp.sum)
    prog.add_fence()
    plan = lower(prog, Machine([2, 4], gpus_per_node=4), ring=1, stripe=1, pipeline=4)
    ex = Executor(plan, device=0, dtype="f32")        # replaces execute_plan (engine.hpp:127)

Every call goes through libhiccl.so; errors surface as HicclError carrying
the reference's ErrorCode name (types.hpp:50-64).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, Sequence

from . import _native as N

lib = N.lib

ERROR_NAMES = ["Ok", "EmptyLeafSet", "RankOutOfRange", "EmptyStep", "WriteWriteRace",
               "ReadWriteRace", "BadBufferRef", "UnsupportedFormulation", "InvalidMachine",
               "InvalidConfig", "UninitializedRead", "DependencyViolation", "NoInterNodeBound",
               "ParseError", "CudaError", "Timeout"]


class HicclError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERROR_NAMES[status] if 0 <= status < len(ERROR_NAMES) else "Internal"
        super().__init__(message)


def _check(status: int) -> None:
    if status != 0:
        raise HicclError(status, lib.hc_last_error().decode())


def _take_string(ptr: C.c_void_p) -> str:
    s = C.string_at(ptr).decode()
    lib.hc_free(ptr)
    return s


class ReduceOp(enum.IntEnum):
    sum = 0
    max = 1


class CollectiveKind(enum.IntEnum):
    scatter = 0
    broadcast = 1
    gather = 2
    reduce = 3
    all_to_all = 4
    all_gather = 5
    reduce_scatter = 6
    all_reduce = 7


class Formulation(enum.IntEnum):
    single = 0
    multi = 1
    multi_alt = 2


DTYPES = {"f32": 0, "bf16": 1, "f16": 2, "i32": 3, "i64": 4, "f64": 5, "u8": 6}
COPY_MODES = {"pull": 0, "push": 1, "staged": 2, "ll": 3, "auto": 4}
ELEMENT_SIZE = {"f32": 4, "bf16": 2, "f16": 2, "i32": 4, "i64": 8, "f64": 8, "u8": 1}


@dataclass(frozen=True)
class BufferRef:
    """types.hpp:36-48"""
    buffer: str
    offset: int
    count: int


@dataclass
class Violation:
    code: str
    step: int
    primitive: int
    rank: int
    buffer: str
    lo: int
    hi: int
    message: str


def _ints(xs: Iterable[int]):
    xs = list(xs)
    return (C.c_int * max(1, len(xs)))(*xs), len(xs)


class CollectiveProgram:
    """composition.hpp:66-122"""

    def __init__(self, world_size: int | None = None, *, _handle=None):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            _check(lib.hc_program_create(world_size, C.byref(self._h)))

    def __del__(self):
        try:
            if getattr(self, "_h", None) and self._h.value:
                lib.hc_program_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:  # interpreter shutdown
            pass

    def declare_buffer(self, name: str, length: int, input: bool = False,
                       internal: bool = False) -> "CollectiveProgram":
        _check(lib.hc_program_declare_buffer(self._h, name.encode(), length, int(input),
                                             int(internal)))
        return self

    def add_multicast(self, send: BufferRef, recv: BufferRef, root: int,
                      leaves: Sequence[int]) -> "CollectiveProgram":
        if send.count != recv.count:
            raise HicclError(6, "BadBufferRef: send.count != recv.count")
        arr, n = _ints(leaves)
        _check(lib.hc_program_add_multicast(self._h, send.buffer.encode(), send.offset,
                                            recv.buffer.encode(), recv.offset, send.count, root,
                                            arr, n))
        return self

    def add_reduction(self, send: BufferRef, recv: BufferRef, leaves: Sequence[int], root: int,
                      op: ReduceOp = ReduceOp.sum) -> "CollectiveProgram":
        if send.count != recv.count:
            raise HicclError(6, "BadBufferRef: send.count != recv.count")
        arr, n = _ints(leaves)
        _check(lib.hc_program_add_reduction(self._h, send.buffer.encode(), send.offset,
                                            recv.buffer.encode(), recv.offset, send.count, arr, n,
                                            root, int(op)))
        return self

    def add_fence(self) -> "CollectiveProgram":
        _check(lib.hc_program_add_fence(self._h))
        return self

    def validate(self) -> list[Violation]:
        out = C.c_void_p()
        _check(lib.hc_program_validate(self._h, C.byref(out)))
        vs = []
        for line in _take_string(out).splitlines():
            code, step, prim, rank, buf, lo, hi, msg = line.split("|", 7)
            vs.append(Violation(code, int(step), int(prim), int(rank), buf, int(lo), int(hi), msg))
        return vs

    def serialize(self) -> str:
        out = C.c_void_p()
        _check(lib.hc_program_serialize(self._h, C.byref(out)))
        return _take_string(out)

    @staticmethod
    def deserialize(text: str) -> "CollectiveProgram":
        h = C.c_void_p()
        _check(lib.hc_program_deserialize(text.encode(), C.byref(h)))
        return CollectiveProgram(_handle=h)

    def id(self) -> str:
        out = C.c_void_p()
        _check(lib.hc_program_id(self._h, C.byref(out)))
        return _take_string(out)


@dataclass
class CollectiveSpec:
    """presets.hpp:53-59"""
    kind: CollectiveKind = CollectiveKind.broadcast
    formulation: Formulation = Formulation.single
    root: int = 0
    count: int = 1
    op: ReduceOp = ReduceOp.sum


def build(spec: CollectiveSpec, p: int) -> CollectiveProgram:
    """presets::build (presets.hpp:62)"""
    h = C.c_void_p()
    _check(lib.hc_program_preset(int(spec.kind), int(spec.formulation), p, spec.count, spec.root,
                                 int(spec.op), C.byref(h)))
    return CollectiveProgram(_handle=h)


def preset_lengths(spec: CollectiveSpec, p: int) -> tuple[int, int]:
    """(sendbuf, recvbuf) element counts of a preset (presets.cpp:116-226)."""
    d = spec.count
    send = d if spec.kind in (CollectiveKind.gather, CollectiveKind.all_gather) else p * d
    recv = d if spec.kind == CollectiveKind.scatter else p * d
    return send, recv


@dataclass
class Machine:
    """MachineDescriptor (machine.hpp:48-89) as far as lowering needs it:
    hierarchy factors, gpus_per_node (g) and the per-level library."""
    hierarchy: list[int]
    gpus_per_node: int = 0  # 0 = p (one node)
    library: list[str] | None = None

    def _desc(self):
        h, n = _ints(self.hierarchy)
        p = 1
        for x in self.hierarchy:
            p *= x
        libs = None
        keep = [h]
        if self.library:
            libs = (C.c_char_p * n)(*[s.encode() for s in self.library])
            keep.append(libs)
        d = N.MachineDesc(h, n, self.gpus_per_node or p, libs)
        return d, keep


class Plan:
    """A PipelinedPlan (pipeline.hpp:31-38)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        info = N.PlanInfo()
        _check(lib.hc_plan_get_info(self._h, C.byref(info)))
        self.world_size = info.world_size
        self.num_transfers = info.num_transfers
        self.num_stages = info.num_stages
        self.slots = info.slots
        self.depth = info.depth
        self.stripe = info.stripe
        self.ring = info.ring
        self.buffers: list[tuple[str, int, bool, bool]] = []
        for i in range(info.num_buffers):
            name = C.c_char_p()
            length = C.c_int64()
            inp = C.c_int()
            internal = C.c_int()
            _check(lib.hc_plan_get_buffer(self._h, i, C.byref(name), C.byref(length),
                                          C.byref(inp), C.byref(internal)))
            self.buffers.append((name.value.decode(), length.value, bool(inp.value),
                                 bool(internal.value)))

    def __del__(self):
        try:
            if getattr(self, "_h", None) and self._h.value:
                lib.hc_plan_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:  # interpreter shutdown
            pass

    @property
    def buffer_names(self) -> list[str]:
        return [b[0] for b in self.buffers]

    def transfers(self):
        arr = (N.Transfer * max(1, self.num_transfers))()
        _check(lib.hc_plan_get_transfers(self._h, arr))
        return arr, self.num_transfers

    def transfer_dicts(self) -> list[dict]:
        arr, n = self.transfers()
        names = self.buffer_names
        out = []
        for k in range(n):
            t = arr[k]
            out.append(dict(id=t.id, src=t.src, dst=t.dst, src_buffer=names[t.src_buf],
                            dst_buffer=names[t.dst_buf], src_offset=t.src_off,
                            dst_offset=t.dst_off, count=t.count, reduce=bool(t.reduce), op=t.op,
                            stage=t.stage, slot=t.slot, channel=t.channel, stripe=t.stripe,
                            level=t.level, step=t.step))
        return out

    def serialize(self) -> str:
        out = C.c_void_p()
        _check(lib.hc_plan_serialize(self._h, C.byref(out)))
        return _take_string(out)

    @staticmethod
    def deserialize(text: str) -> "Plan":
        h = C.c_void_p()
        _check(lib.hc_plan_deserialize(text.encode(), C.byref(h)))
        return Plan(h)

    def schedule_summary(self, num_execs: int = 1, rank_to_exec: Sequence[int] | None = None,
                         copy_mode: str = "pull", element_size: int = 4,
                         verify: bool = True) -> dict:
        import json
        r2e = rank_to_exec if rank_to_exec is not None else split_ranks(self.world_size, num_execs)
        arr, _ = _ints(r2e)
        out = C.c_void_p()
        _check(lib.hc_plan_schedule_summary(self._h, num_execs, arr, COPY_MODES[copy_mode],
                                            element_size, int(verify), C.byref(out)))
        return json.loads(_take_string(out))

    def layout_summary(self, num_execs: int = 1, rank_to_exec: Sequence[int] | None = None,
                       copy_mode: str = "push", dtype: str = "f32", ctas: int = 0,
                       multicast: Sequence[str] = ()) -> dict:
        """Device items per executor and step as the executors would build
        them with `multicast` buffers in an NVLS window (multimem lowering and
        reduce+multicast fusion), tile hazards verified pair by pair."""
        import json
        r2e = rank_to_exec if rank_to_exec is not None else split_ranks(self.world_size, num_execs)
        arr, _ = _ints(r2e)
        out = C.c_void_p()
        _check(lib.hc_plan_layout_summary(self._h, num_execs, arr, COPY_MODES[copy_mode],
                                          DTYPES[dtype], ctas, ",".join(multicast).encode(),
                                          C.byref(out)))
        return json.loads(_take_string(out))

    def comm_matrix(self, slot: int) -> list[list[int]]:
        p = self.world_size
        out = (C.c_int64 * (p * p))()
        _check(lib.hc_plan_comm_matrix(self._h, slot, out))
        return [[out[i * p + j] for j in range(p)] for i in range(p)]


def lower(program: CollectiveProgram, machine: Machine, ring: int = 1, stripe: int = 1,
          pipeline: int = 1) -> Plan:
    """lower() + pipeline() (factorize.hpp:107-109, pipeline.hpp:40); argument
    order of the paper's init(hierarchy, library, ring, stripe, pipeline)."""
    desc, keep = machine._desc()
    h = C.c_void_p()
    _check(lib.hc_plan_lower(program._h, C.byref(desc), ring, stripe, pipeline, C.byref(h)))
    del keep
    return Plan(h)


def lower_staged_json(program: CollectiveProgram, machine: Machine, ring: int = 1,
                      stripe: int = 1) -> str:
    desc, keep = machine._desc()
    out = C.c_void_p()
    _check(lib.hc_plan_lower_staged_json(program._h, C.byref(desc), ring, stripe, C.byref(out)))
    del keep
    return _take_string(out)


class PlanCache:
    """Persistent plans (the paper's init-once design):
    lower() + pipeline() memoized in memory and, with `directory`, on disk
    as hiercoll-pipelined-v1 JSON keyed by (program id, machine, ring,
    stripe, pipeline). A cached plan deserializes into the same plan the
    factorizer would build (serialization is byte-identical)."""

    def __init__(self, directory: str | None = None):
        import os
        self.directory = directory
        self._mem: dict[str, str] = {}
        self.hits = self.misses = 0
        if directory:
            os.makedirs(directory, exist_ok=True)

    @staticmethod
    def key(program: CollectiveProgram, machine: Machine, ring: int, stripe: int,
            pipeline: int) -> str:
        import hashlib
        text = "|".join([program.id(), ",".join(map(str, machine.hierarchy)),
                         str(machine.gpus_per_node), ",".join(machine.library or []),
                         str(ring), str(stripe), str(pipeline)])
        return hashlib.sha256(text.encode()).hexdigest()[:32]

    def lower(self, program: CollectiveProgram, machine: Machine, ring: int = 1,
              stripe: int = 1, pipeline: int = 1) -> "Plan":
        import os
        k = self.key(program, machine, ring, stripe, pipeline)
        text = self._mem.get(k)
        path = os.path.join(self.directory, k + ".json") if self.directory else None
        if text is None and path and os.path.exists(path):
            with open(path) as f:
                text = f.read()
        if text is not None:
            self.hits += 1
            self._mem[k] = text
            return Plan.deserialize(text)
        self.misses += 1
        plan = lower(program, machine, ring=ring, stripe=stripe, pipeline=pipeline)
        text = plan.serialize()
        self._mem[k] = text
        if path:
            tmp = path + ".tmp%d" % os.getpid()
            with open(tmp, "w") as f:
                f.write(text)
            os.replace(tmp, path)
        return plan


# --------------------------------------------------------------------- model

def default_model() -> dict:
    m = N.Model()
    _check(lib.hc_model_default(C.byref(m)))
    return {f: getattr(m, f) for f, _ in N.Model._fields_}


def _model(model: dict | None):
    if model is None:
        return None
    m = N.Model()
    base = default_model()
    base.update(model)
    for k, v in base.items():
        setattr(m, k, v)
    return C.byref(m)


def predict(plan: "Plan", element_size: int = 4, model: dict | None = None,
            ranks_per_gpu: int = 1, copy_mode: str = "push") -> float:
    """Modelled seconds of one execution (include/hiccl/model.hpp)."""
    out = C.c_double()
    _check(lib.hc_plan_predict(plan._h, element_size, _model(model), ranks_per_gpu,
                               COPY_MODES[copy_mode], C.byref(out)))
    return out.value


def tune(kind: CollectiveKind, p: int, count: int, element_size: int = 4,
         model: dict | None = None) -> dict:
    """Model-best formulation / ring / pipeline depth / copy mode for a preset
    on flat {p} (ring > 1 means a g = 1 machine description)."""
    r = N.TuneResult()
    _check(lib.hc_tune(int(kind), p, count, element_size, _model(model), C.byref(r)))
    mode = {v: k for k, v in COPY_MODES.items()}[r.copy_mode]
    return {"formulation": Formulation(r.formulation), "ring": r.ring, "pipeline": r.pipeline,
            "seconds": r.seconds, "copy_mode": mode}


def predict_nvls(plan: "Plan", dtype: str = "f32", model: dict | None = None) -> float:
    """Modelled seconds with the user buffers in an NVLS window."""
    out = C.c_double()
    _check(lib.hc_plan_predict_nvls(plan._h, DTYPES[dtype], _model(model), C.byref(out)))
    return out.value


def tune_nvls(kind: CollectiveKind, p: int, count: int, dtype: str = "f32",
              model: dict | None = None) -> dict:
    """tune(), also weighing the NVLS library ("nvls": True when it wins)."""
    r = N.TuneResult()
    _check(lib.hc_tune_nvls(int(kind), p, count, DTYPES[dtype], _model(model), C.byref(r)))
    mode = {v: k for k, v in COPY_MODES.items()}[r.copy_mode]
    return {"formulation": Formulation(r.formulation), "ring": r.ring, "pipeline": r.pipeline,
            "seconds": r.seconds, "copy_mode": mode, "nvls": bool(r.nvls)}


def t_ring(alpha, d, k, f, m, n, intra=0.0) -> float:
    out = C.c_double()
    _check(lib.hc_t_ring(alpha, d, k, f, m, n, intra, C.byref(out)))
    return out.value


def t_tree(alpha, d, k, f, m, n, intra=0.0) -> float:
    out = C.c_double()
    _check(lib.hc_t_tree(alpha, d, k, f, m, n, intra, C.byref(out)))
    return out.value


def bound(kind: CollectiveKind, p: int, g: int, k: int, f: float) -> float:
    out = C.c_double()
    _check(lib.hc_bound(int(kind), p, g, k, f, C.byref(out)))
    return out.value


def throughput(d_bytes: float, p: int, t: float) -> float:
    out = C.c_double()
    _check(lib.hc_throughput(d_bytes, p, t, C.byref(out)))
    return out.value


# --------------------------------------------------------------------- devices

def device_count() -> int:
    n = C.c_int()
    _check(lib.hc_device_count(C.byref(n)))
    return n.value


def enable_peer_access(devices: Sequence[int]) -> None:
    arr, n = _ints(devices)
    _check(lib.hc_enable_peer_access(arr, n))


def device_fill(device: int, ptr: int, count: int, dtype: str, seed: int, rank: int,
                index_base: int = 0, stream: int = 0) -> None:
    _check(lib.hc_device_fill(device, C.c_void_p(ptr), count, DTYPES[dtype], seed, rank,
                              index_base, C.c_void_p(stream)))


def ipc_export(ptr: int) -> tuple[bytes, int]:
    h = (C.c_ubyte * 64)()
    off = C.c_size_t()
    _check(lib.hc_ipc_export(C.c_void_p(ptr), h, C.byref(off)))
    return bytes(h), off.value


def ipc_import(handle: bytes, offset: int, device: int) -> int:
    h = (C.c_ubyte * 64)(*handle)
    out = C.c_void_p()
    _check(lib.hc_ipc_import(h, offset, device, C.byref(out)))
    return out.value


def nvls_supported(device: int = 0) -> bool:
    s = C.c_int()
    _check(lib.hc_nvls_supported(device, C.byref(s)))
    return bool(s.value)


class DeviceView:
    """A raw device range as a __cuda_array_interface__ object (torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


class Window:
    """NVLS window: symmetric device memory bound to an NVSwitch multicast
    object (hc_window_*). Single-process form spans `devices`."""

    def __init__(self, devices: Sequence[int] | None = None, nbytes: int = 0, *, _handle=None,
                 members: int = 0):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
            self.members = members
        else:
            arr, n = _ints(devices)
            _check(lib.hc_window_create(arr, n, nbytes, C.byref(self._h)))
            self.members = n

    @staticmethod
    def open(device: int, n_members: int, nbytes: int, handle: bytes | None) -> "Window":
        h = C.c_void_p()
        hb = (C.c_ubyte * 64)(*handle) if handle else None
        _check(lib.hc_window_open(device, n_members, nbytes, hb, C.byref(h)))
        return Window(_handle=h, members=1)

    def export(self) -> bytes:
        h = (C.c_ubyte * 64)()
        _check(lib.hc_window_export(self._h, h))
        return bytes(h)

    def bind(self) -> None:
        _check(lib.hc_window_bind(self._h))

    def export_memory(self) -> bytes:
        h = (C.c_ubyte * 64)()
        _check(lib.hc_window_export_memory(self._h, h))
        return bytes(h)

    def import_memory(self, handle: bytes) -> int:
        out = C.c_void_p()
        _check(lib.hc_window_import_memory(self._h, (C.c_ubyte * 64)(*handle), C.byref(out)))
        return out.value

    def pointers(self, member: int = 0) -> tuple[int, int, int]:
        uc, mc, n = C.c_void_p(), C.c_void_p(), C.c_size_t()
        _check(lib.hc_window_pointers(self._h, member, C.byref(uc), C.byref(mc), C.byref(n)))
        return uc.value, mc.value, n.value

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib.hc_window_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def window_layout(sizes: dict[str, int], align: int = 1 << 21) -> tuple[dict[str, int], int]:
    """Offsets of named buffers inside a window (2 MiB aligned)."""
    off, out = 0, {}
    for name, n in sizes.items():
        out[name] = off
        off += (n + align - 1) // align * align
    return out, max(off, align)


class Executor:
    """One persistent sm_100a executor (one GPU) serving the ranks mapped to it.
    Replaces execute_plan/run_transfers (engine.hpp:127, engine.cpp:285-347)."""

    def __init__(self, plan: Plan, device: int = 0, exec_index: int = 0, num_execs: int = 1,
                 rank_to_exec: Sequence[int] | None = None, dtype: str = "f32", ctas: int = 0,
                 threads: int = 0, copy_mode: str = "push", timeout_s: float = 30.0,
                 execs_per_device: int = 1):
        self.plan = plan
        self.device = device
        self.exec_index = exec_index
        self.num_execs = num_execs
        self.dtype = dtype
        if rank_to_exec is None:
            rank_to_exec = [0] * plan.world_size
        self.rank_to_exec = list(rank_to_exec)
        r2e, _ = _ints(self.rank_to_exec)
        cfg = N.ExecConfig(device, exec_index, num_execs, r2e, DTYPES[dtype], ctas, threads,
                           COPY_MODES[copy_mode], timeout_s, execs_per_device)
        self._h = C.c_void_p()
        _check(lib.hc_exec_create(plan._h, C.byref(cfg), C.byref(self._h)))

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib.hc_exec_destroy(self._h)
            self._h = C.c_void_p()

    def bind_buffer(self, rank: int, name: str, ptr: int, nbytes: int) -> None:
        _check(lib.hc_exec_bind_buffer(self._h, rank, name.encode(), C.c_void_p(ptr), nbytes))

    def bind_multicast(self, name: str, mc_ptr: int) -> None:
        _check(lib.hc_exec_bind_multicast(self._h, name.encode(), C.c_void_p(mc_ptr)))

    def local_arena(self) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_size_t()
        _check(lib.hc_exec_local_arena(self._h, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def bind_peer_arena(self, peer: int, ptr: int) -> None:
        _check(lib.hc_exec_bind_peer_arena(self._h, peer, C.c_void_p(ptr)))

    def local_flags(self) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_size_t()
        _check(lib.hc_exec_local_flags(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def bind_peer_flags(self, peer: int, ptr: int) -> None:
        _check(lib.hc_exec_bind_peer_flags(self._h, peer, C.c_void_p(ptr)))

    def commit(self) -> None:
        _check(lib.hc_exec_commit(self._h))

    def start(self, stream: int = 0) -> None:
        _check(lib.hc_exec_start(self._h, C.c_void_p(stream)))

    def wait(self) -> None:
        _check(lib.hc_exec_wait(self._h))

    def query(self) -> bool:
        d = C.c_int()
        _check(lib.hc_exec_query(self._h, C.byref(d)))
        return bool(d.value)

    def trace(self) -> dict:
        """Device timeline of the last launch in microseconds from grid entry."""
        S = self.stats()["num_steps"]
        n = S + 4
        arr = (C.c_int64 * (n + 128))()
        _check(lib.hc_exec_get_trace(self._h, arr, n + 128))
        t0 = arr[0]
        rel = lambda v: (v - t0) / 1e3 if v >= t0 and v > 0 else None
        out = {"entry_barrier_us": rel(arr[1]),
               "steps_us": [rel(arr[2 + s]) for s in range(S)],
               "last_cta_us": rel(arr[n - 2]), "exit_us": rel(arr[n - 1])}
        warps = []  # tagged-line mode: CTA 0's per-warp [start, end] per step
        for s in range(min(S, 4)):
            row = [(rel(arr[n + (s * 16 + w) * 2]), rel(arr[n + (s * 16 + w) * 2 + 1]))
                   for w in range(16)]
            if any(a is not None for a, _ in row):
                warps.append(row)
        if warps:
            out["warps_us"] = warps
        return out

    def stats(self) -> dict:
        s = N.ExecStats()
        _check(lib.hc_exec_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in N.ExecStats._fields_}


def split_ranks(world_size: int, num_execs: int) -> list[int]:
    """Contiguous ranks per executor (rank r -> r // (p / E)); p % E == 0."""
    if world_size % num_execs:
        raise HicclError(9, f"InvalidConfig: {world_size} ranks do not split over {num_execs} GPUs")
    per = world_size // num_execs
    return [r // per for r in range(world_size)]


class World:
    """Single-process driver: one Executor per device, peer access enabled,
    arenas and flag words cross-bound directly (no IPC needed)."""

    def __init__(self, plan: Plan, devices: Sequence[int], dtype: str = "f32",
                 rank_to_exec: Sequence[int] | None = None, **exec_kw):
        self.plan = plan
        self.devices = list(devices)
        E = len(self.devices)
        self.rank_to_exec = list(rank_to_exec) if rank_to_exec is not None else \
            split_ranks(plan.world_size, E)
        if len(set(self.devices)) > 1:
            enable_peer_access(sorted(set(self.devices)))
        # several executors may share a GPU (each then runs on its own
        # stream with 1/n of the device's CTAs): the cross-executor protocol
        # is the same as between GPUs, so a one-GPU box exercises it too
        share = max(self.devices.count(d) for d in self.devices)
        exec_kw.setdefault("execs_per_device", share)
        self.execs = [Executor(plan, device=d, exec_index=i, num_execs=E,
                               rank_to_exec=self.rank_to_exec, dtype=dtype, **exec_kw)
                      for i, d in enumerate(self.devices)]
        arenas = [e.local_arena()[0] for e in self.execs]
        flags = [e.local_flags()[0] for e in self.execs]
        for e in self.execs:
            for j in range(E):
                if j != e.exec_index:
                    e.bind_peer_arena(j, arenas[j])
                    e.bind_peer_flags(j, flags[j])

    def device_of(self, rank: int) -> int:
        return self.devices[self.rank_to_exec[rank]]

    def enable_nvls(self, sizes: dict[str, int]) -> dict[tuple[int, str], int]:
        """Place user buffers `name -> bytes` of every rank in one NVLS window
        (one rank per GPU) and bind them; returns (rank, name) -> device
        address for the caller to fill / read."""
        if len(set(self.devices)) != len(self.devices) or self.plan.world_size != len(self.devices):
            raise HicclError(9, "InvalidConfig: NVLS needs one rank per GPU")
        offs, total = window_layout(sizes)
        self.window = Window(self.devices, total)
        where = {}
        for i, e in enumerate(self.execs):
            uc, mc, _ = self.window.pointers(i)
            for name, off in offs.items():
                e.bind_multicast(name, mc + off)
        for r in range(self.plan.world_size):
            uc, _, _ = self.window.pointers(self.rank_to_exec[r])
            for name, off in offs.items():
                self.bind(r, name, uc + off, sizes[name])
                where[(r, name)] = uc + off
        return where

    def bind(self, rank: int, name: str, ptr: int, nbytes: int) -> None:
        for e in self.execs:
            e.bind_buffer(rank, name, ptr, nbytes)

    def commit(self) -> None:
        for e in self.execs:
            e.commit()

    def start(self, streams: Sequence[int] | None = None) -> None:
        for i, e in enumerate(self.execs):
            e.start(streams[i] if streams else 0)

    def wait(self) -> None:
        for e in self.execs:
            e.wait()

    def run(self) -> None:
        self.start()
        self.wait()

    def close(self) -> None:
        # every grid must be finished before any executor's memory goes:
        # a peer still running (e.g. after another executor failed) writes
        # into this executor's flag words and reads its arena
        for e in self.execs:
            try:
                e.wait()
            except HicclError:
                pass
        for e in self.execs:
            e.close()
        if getattr(self, "window", None) is not None:
            self.window.close()
            self.window = None
