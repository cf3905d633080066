"""TEST INFRASTRUCTURE — the parity oracle. Never imported by the product.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker.

Two checkers live here:

* ``Reference`` — the UNMODIFIED reference library (``hiercoll``) compiled
  from /root/reference/proj/src into oracle/_ref/libhiercoll_ref.so by
  oracle/Makefile, driven through oracle/ref_driver.cpp. It produces the
  reference's own plans (factorize.cpp:587, pipeline.cpp:76) and runs its
  symbolic executor + ground truth (engine.cpp:285-347, presets.cpp:231,
  engine.cpp:221). That pins *dataflow* exactly.
* ``numeric`` — oracle/numeric_exec.c, a C restatement of the reference
  executor's transfer loop (engine.cpp:285-330) on numbers, with the fold
  rules stated in its header. Numeric results are "parity unpinned" by the
  reference itself (it is symbolic only); the restatement is
  pinned instead by (a) integer inputs, where any fold order must give the
  exact ground-truth sum/max computed independently here, and (b) running
  it on the reference's own plans.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "liboracle_exec.so"
REF_LIB = HERE / "_ref" / "libhiercoll_ref.so"

DTYPES = {"f32": (0, np.float32), "bf16": (1, np.uint16), "f16": (2, np.uint16),
          "i32": (3, np.int32), "i64": (4, np.int64), "f64": (5, np.float64), "u8": (6, np.uint8)}


class Transfer(C.Structure):  # same layout as or_transfer in numeric_exec.c
    _fields_ = [(n, C.c_int32) for n in ("id", "src", "dst", "src_buf", "dst_buf", "reduce", "op",
                                         "stage", "slot", "channel", "stripe", "level", "step",
                                         "n_deps")] + \
               [(n, C.c_int64) for n in ("src_off", "dst_off", "count")]


_port = None


def port():
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            raise ImportError(f"{PORT_LIB} missing: run `make -C oracle port`")
        lib = C.CDLL(str(PORT_LIB))
        lib.oracle_fill.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int64]
        lib.oracle_fill.restype = None
        lib.oracle_run_transfers.argtypes = [C.POINTER(Transfer), C.c_int, C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_int64), C.c_int, C.c_int, C.c_int,
                                             C.POINTER(C.c_void_p), C.c_int]
        lib.oracle_run_transfers.restype = C.c_int
        _port = lib
    return _port


def fill(n: int, dtype: str, seed: int, rank: int, index_base: int = 0) -> np.ndarray:
    """The shared counter-hash generator (numeric_exec.c header)."""
    code, npdt = DTYPES[dtype]
    out = np.empty(n, dtype=npdt)
    port().oracle_fill(out.ctypes.data, n, code, seed, rank, index_base)
    return out


SENTINEL_SEED = 0x5E471E1


def sentinel(n: int, dtype: str, rank: int) -> np.ndarray:
    """Pre-fill for non-input buffers (catches unwritten elements)."""
    return fill(n, dtype, SENTINEL_SEED, rank)


# ---------------------------------------------------------------- plans

class FlatPlan:
    """A pipelined plan as the oracle consumes it: buffers (name order) and
    transfers in id order."""

    def __init__(self, world_size: int, buffers: list[tuple[str, int, bool, bool]],
                 transfers: list[dict]):
        self.world_size = world_size
        self.buffers = buffers
        self.names = [b[0] for b in buffers]
        self.transfers = transfers

    @staticmethod
    def from_json(text: str) -> "FlatPlan":
        j = json.loads(text)
        bufs = [(b["id"], b["length"], b["input"], b["internal"]) for b in j["buffers"]]
        ts = []
        for t in j["transfers"]:
            ts.append(dict(id=t["id"], src=t["src"], dst=t["dst"], src_buffer=t["src_buffer"],
                           dst_buffer=t["dst_buffer"], src_offset=t["src_offset"],
                           dst_offset=t["dst_offset"], count=t["count"],
                           reduce=t["op"] != "copy", op=1 if t["op"] == "max" else 0,
                           stage=t["stage"], slot=t["slot"], channel=t["channel"],
                           stripe=t["stripe"], level=t["level"], step=t["step"]))
        return FlatPlan(j["world_size"], bufs, ts)

    @staticmethod
    def from_dicts(world_size: int, buffers, transfers: list[dict]) -> "FlatPlan":
        return FlatPlan(world_size, list(buffers), list(transfers))


def execute(plan: FlatPlan, dtype: str, state: dict[str, list[np.ndarray]], threads: int = 1,
            track_defined: bool = False) -> dict[str, list[np.ndarray]]:
    """Run the restated reference executor in place over ``state``
    (buffer name -> per-rank arrays). Internal buffers missing from
    ``state`` are allocated (zero) at full declared length."""
    code, npdt = DTYPES[dtype]
    p = plan.world_size
    nb = len(plan.names)
    for name, length, _inp, internal in plan.buffers:
        if name not in state:
            state[name] = [np.zeros(length, dtype=npdt) for _ in range(p)]
    ptrs = (C.c_void_p * (nb * p))()
    lengths = (C.c_int64 * nb)()
    defined = None
    keep = []
    if track_defined:
        defined = (C.c_void_p * (nb * p))()
    for b, (name, length, inp, internal) in enumerate(plan.buffers):
        lengths[b] = length
        for r in range(p):
            arr = state[name][r]
            assert arr.dtype == npdt and arr.size >= length and arr.flags.c_contiguous
            ptrs[b * p + r] = arr.ctypes.data
            if track_defined:
                d = np.full(length, 1 if inp else 0, dtype=np.uint8)
                keep.append(d)
                defined[b * p + r] = d.ctypes.data
    idx = {n: i for i, n in enumerate(plan.names)}
    ts = (Transfer * max(1, len(plan.transfers)))()
    for k, t in enumerate(plan.transfers):
        x = ts[k]
        x.id, x.src, x.dst = t["id"], t["src"], t["dst"]
        x.src_buf, x.dst_buf = idx[t["src_buffer"]], idx[t["dst_buffer"]]
        x.reduce, x.op, x.stage, x.slot = int(t["reduce"]), t["op"], t["stage"], t["slot"]
        x.src_off, x.dst_off, x.count = t["src_offset"], t["dst_offset"], t["count"]
    rc = port().oracle_run_transfers(ts, len(plan.transfers), ptrs, lengths, p, nb, code,
                                     defined, threads)
    if rc == 10:
        raise RuntimeError("UninitializedRead in plan replay")
    if rc:
        raise RuntimeError(f"oracle_run_transfers failed with {rc}")
    return state


# ---------------------------------------------------------------- reference library

class Reference:
    """The compiled reference library (oracle/_ref)."""

    def __init__(self, path: Path = REF_LIB):
        if not path.exists():
            raise ImportError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(str(path))
        P, cp, i = C.POINTER, C.c_char_p, C.c_int
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_program_json.argtypes = [i, i, i, C.c_int64, i, i, P(C.c_void_p), P(C.c_void_p)]
        L.ref_preset_pipelined_json.argtypes = [i, i, i, C.c_int64, i, i, P(i), i, i, i, i, i,
                                                P(C.c_void_p), P(C.c_void_p)]
        L.ref_preset_staged_json.argtypes = [i, i, i, C.c_int64, i, i, P(i), i, i, i, i,
                                             P(C.c_void_p), P(C.c_void_p)]
        L.ref_lower_program_json.argtypes = [cp, P(i), i, i, i, i, i, P(C.c_void_p), P(C.c_void_p)]
        L.ref_roundtrip_program_json.argtypes = [cp, P(C.c_void_p), P(C.c_void_p)]
        L.ref_validate_program_json.argtypes = [cp, P(C.c_void_p), P(C.c_void_p)]
        L.ref_check_pipelined_json.argtypes = [cp, i, i, i, C.c_int64, i, i, P(C.c_void_p),
                                               P(C.c_void_p)]
        L.ref_check_program_plan.argtypes = [cp, cp, P(C.c_void_p), P(C.c_void_p)]
        L.ref_time_execute_plan.argtypes = [i, i, i, C.c_int64, i, i, P(i), i, i, i, i, i,
                                            P(C.c_double), P(C.c_void_p)]
        L.ref_simulate_seconds.argtypes = [cp, P(i), i, i, P(C.c_double), P(C.c_void_p)]
        L.ref_inter_node_bytes.argtypes = [cp, i, P(C.c_int64), P(C.c_void_p)]
        self.L = L

    def _s(self, ptr: C.c_void_p) -> str:
        if not ptr.value:
            return ""
        s = C.string_at(ptr).decode()
        self.L.ref_free(ptr)
        return s

    def _call(self, fn, *args):
        out, err = C.c_void_p(), C.c_void_p()
        rc = fn(*args, C.byref(out), C.byref(err))
        return rc, self._s(out), self._s(err)

    @staticmethod
    def _h(hier):
        return (C.c_int * len(hier))(*hier), len(hier)

    def program_json(self, kind, form, p, count, root=0, op=0) -> str:
        rc, out, err = self._call(self.L.ref_program_json, kind, form, p, count, root, op)
        if rc:
            raise RuntimeError(err)
        return out

    def preset_plan(self, kind, form, p, count, root, op, hier, g, stripe, ring, depth):
        """(rc, pipelined-plan JSON or error text)"""
        h, n = self._h(hier)
        rc, out, err = self._call(self.L.ref_preset_pipelined_json, kind, form, p, count, root,
                                  op, h, n, g, stripe, ring, depth)
        return (rc, out) if rc == 0 else (rc, err)

    def preset_staged(self, kind, form, p, count, root, op, hier, g, stripe, ring):
        h, n = self._h(hier)
        rc, out, err = self._call(self.L.ref_preset_staged_json, kind, form, p, count, root, op,
                                  h, n, g, stripe, ring)
        return (rc, out) if rc == 0 else (rc, err)

    def lower_program(self, program_json: str, hier, g, stripe, ring, depth):
        h, n = self._h(hier)
        rc, out, err = self._call(self.L.ref_lower_program_json, program_json.encode(), h, n, g,
                                  stripe, ring, depth)
        return (rc, out) if rc == 0 else (rc, err)

    def roundtrip_program(self, program_json: str) -> str:
        rc, out, err = self._call(self.L.ref_roundtrip_program_json, program_json.encode())
        if rc:
            raise RuntimeError(err)
        return out

    def validate_program(self, program_json: str) -> list[str]:
        rc, out, err = self._call(self.L.ref_validate_program_json, program_json.encode())
        if rc:
            raise RuntimeError(err)
        return [line.split("|")[0] for line in out.splitlines()]

    def check_plan(self, plan_json: str, kind, form, p, count, root=0, op=0) -> tuple[int, str]:
        """0 = PASS; 1 = divergence (message); >1 = error."""
        rc, out, err = self._call(self.L.ref_check_pipelined_json, plan_json.encode(), kind, form,
                                  p, count, root, op)
        return rc, out or err

    def check_program_plan(self, program_json: str, plan_json: str) -> tuple[int, str]:
        rc, out, err = self._call(self.L.ref_check_program_plan, program_json.encode(),
                                  plan_json.encode())
        return rc, out or err

    def time_execute_plan(self, kind, form, p, count, root, op, hier, g, stripe, ring,
                          depth) -> float:
        h, n = self._h(hier)
        secs, err = C.c_double(), C.c_void_p()
        rc = self.L.ref_time_execute_plan(kind, form, p, count, root, op, h, n, g, stripe, ring,
                                          depth, C.byref(secs), C.byref(err))
        if rc:
            raise RuntimeError(self._s(err))
        return secs.value

    def simulate(self, plan_json: str, hier, g) -> float:
        h, n = self._h(hier)
        secs, err = C.c_double(), C.c_void_p()
        rc = self.L.ref_simulate_seconds(plan_json.encode(), h, n, g, C.byref(secs), C.byref(err))
        if rc:
            raise RuntimeError(self._s(err))
        return secs.value

    def inter_node_bytes(self, staged_json: str, node_size: int) -> int:
        b, err = C.c_int64(), C.c_void_p()
        rc = self.L.ref_inter_node_bytes(staged_json.encode(), node_size, C.byref(b),
                                         C.byref(err))
        if rc:
            raise RuntimeError(self._s(err))
        return b.value


def reference_available() -> bool:
    return REF_LIB.exists()


# ---------------------------------------------------------------- ground truth

def ground_truth(kind: int, p: int, d: int, root: int, op: int, dtype: str,
                 sends: list[np.ndarray], recv_init: list[np.ndarray]) -> list[np.ndarray]:
    """Standard collective semantics on numbers (mirrors the symbolic
    reference_semantics, presets.cpp:231-298). Exact for integer dtypes
    under any fold order; the caller uses it for i32/i64/u8 and for max."""
    npdt = DTYPES[dtype][1]
    out = [r.copy() for r in recv_init]
    wide = np.int64 if dtype in ("i32", "i64", "u8") else None

    def red(index_slice):
        stack = np.stack([s[index_slice] for s in sends])
        if op == 1:
            return stack.max(axis=0).astype(npdt)
        acc = stack.astype(wide).sum(axis=0)
        if dtype == "u8":
            return (acc & 0xFF).astype(npdt)
        if dtype == "i32":
            return ((acc + 2**31) % 2**32 - 2**31).astype(npdt)
        return acc.astype(npdt)

    if kind == 0:  # scatter
        for j in range(p):
            out[j][:d] = sends[root][j * d:(j + 1) * d]
    elif kind == 1:  # broadcast
        for r in range(p):
            out[r][:p * d] = sends[root][:p * d]
    elif kind == 2:  # gather
        for i in range(p):
            out[root][i * d:(i + 1) * d] = sends[i][:d]
    elif kind == 3:  # reduce
        out[root][:p * d] = red(slice(0, p * d))
    elif kind == 4:  # all_to_all
        for i in range(p):
            for j in range(p):
                out[j][i * d:(i + 1) * d] = sends[i][j * d:(j + 1) * d]
    elif kind == 5:  # all_gather
        for r in range(p):
            for i in range(p):
                out[r][i * d:(i + 1) * d] = sends[i][:d]
    elif kind == 6:  # reduce_scatter
        for j in range(p):
            out[j][j * d:(j + 1) * d] = red(slice(j * d, (j + 1) * d))
    elif kind == 7:  # all_reduce
        v = red(slice(0, p * d))
        for r in range(p):
            out[r][:p * d] = v
    return out
