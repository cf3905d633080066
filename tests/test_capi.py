"""The C ABI boundary: the library loads on a CPU-only host, exports every
entry point include/hiccl.h declares, maps errors to the reference's
ErrorCode order, and fails loudly (no fallback) when a device is needed."""
import re
import subprocess
from pathlib import Path

import pytest

from paper_2408_05962_b200 import _native as N
from paper_2408_05962_b200 import hiccl as H

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hiccl.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (hc_[a-z0-9_]+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing


def test_bindings_cover_header():
    assert set(declared_symbols()) <= set(N.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_error_codes_follow_reference_order():
    # types.hpp:50-64 order, status = 1 + code
    assert H.ERROR_NAMES[1:14] == ["EmptyLeafSet", "RankOutOfRange", "EmptyStep",
                                   "WriteWriteRace", "ReadWriteRace", "BadBufferRef",
                                   "UnsupportedFormulation", "InvalidMachine", "InvalidConfig",
                                   "UninitializedRead", "DependencyViolation", "NoInterNodeBound",
                                   "ParseError"]
    with pytest.raises(H.HicclError) as e:
        H.build(H.CollectiveSpec(H.CollectiveKind.scatter, H.Formulation.multi), 4)
    assert e.value.code == "UnsupportedFormulation" and e.value.status == 7
    assert "UnsupportedFormulation" in H.lib.hc_last_error().decode()


def test_invalid_machine_and_config():
    prog = H.build(H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, 4), 8)
    with pytest.raises(H.HicclError) as e:
        H.lower(prog, H.Machine([3, 3], 9), 1, 1, 1)
    assert e.value.code == "InvalidMachine"
    with pytest.raises(H.HicclError) as e:
        H.lower(prog, H.Machine([2, 4], 4), ring=3)
    assert e.value.code == "InvalidConfig"
    with pytest.raises(H.HicclError) as e:
        H.lower(prog, H.Machine([2, 4], 4), stripe=8)
    assert e.value.code == "InvalidConfig"
    with pytest.raises(H.HicclError) as e:
        H.lower(prog, H.Machine([2, 4], 4), pipeline=0)
    assert e.value.code == "InvalidConfig"


def test_plan_roundtrip_and_introspection():
    prog = H.build(H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, 10), 4)
    plan = H.lower(prog, H.Machine([2, 2], 2), ring=2, stripe=2, pipeline=3)
    text = plan.serialize()
    back = H.Plan.deserialize(text)
    assert back.serialize() == text
    assert back.num_transfers == plan.num_transfers and back.slots == plan.slots
    ts = plan.transfer_dicts()
    assert [t["id"] for t in ts] == list(range(len(ts)))
    total = sum(sum(sum(r) for r in plan.comm_matrix(s)) for s in range(plan.slots))
    assert total == sum(t["count"] for t in ts) * 4


def test_device_entry_points_fail_loudly_without_gpu():
    if H.device_count() > 0:
        pytest.skip("a GPU is present")
    prog = H.build(H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, 4), 2)
    plan = H.lower(prog, H.Machine([2], 2))
    with pytest.raises(H.HicclError) as e:
        H.Executor(plan, device=0)
    assert e.value.code == "CudaError"
