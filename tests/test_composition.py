"""Composition rules — the reference's own unit tests
(proj/tests/test_composition.cpp:41-191) re-expressed against hiccl's C ABI,
case for case, plus the validate() diagnostics compared with the reference
library on the same programs when it is built."""
import pytest

import oracle
from paper_2408_05962_b200.hiccl import (BufferRef, CollectiveProgram, HicclError, ReduceOp)


def base_program(p, length=16):
    prog = CollectiveProgram(p)
    prog.declare_buffer("sendbuf", length, input=True)
    prog.declare_buffer("recvbuf", length)
    return prog


def codes(vs):
    return {v.code for v in vs}


def steps_of(prog):
    import json
    return json.loads(prog.serialize())["steps"]


def test_broadcast_registration_produces_one_primitive():  # test_composition.cpp:41-50
    prog = base_program(6)
    prog.add_multicast(BufferRef("sendbuf", 0, 8), BufferRef("recvbuf", 0, 8), 0, [0, 1, 2, 3, 4, 5])
    st = steps_of(prog)
    assert sum(len(s) for s in st) == 1
    p = st[0][0]
    assert p["root"] == 0 and p["root_participates"] is True
    assert p["leaves"] == [1, 2, 3, 4, 5]


def test_singleton_leaf_set_is_accepted():  # :52-57
    prog = base_program(6)
    prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [3])
    p = steps_of(prog)[0][0]
    assert p["leaves"] == [3] and p["root_participates"] is False


def test_empty_leaf_set_is_rejected():  # :59-64
    prog = base_program(6)
    with pytest.raises(HicclError) as e:
        prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [])
    assert e.value.code == "EmptyLeafSet" and "EmptyLeafSet" in str(e.value)


def test_out_of_range_ranks_are_rejected():  # :66-73
    prog = base_program(4)
    with pytest.raises(HicclError):
        prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [4])
    with pytest.raises(HicclError):
        prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), -1, [1])


def test_buffer_range_checks():  # :75-83
    prog = base_program(4, 8)
    with pytest.raises(HicclError):
        prog.add_multicast(BufferRef("sendbuf", 4, 8), BufferRef("recvbuf", 0, 8), 0, [1])
    with pytest.raises(HicclError):
        prog.add_multicast(BufferRef("nosuch", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1])
    with pytest.raises(HicclError):
        prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 8), 0, [1])


def test_overlapping_destinations_in_one_step_are_rejected_eagerly():  # :85-93
    prog = base_program(6)
    prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1, 2])
    with pytest.raises(HicclError) as e:
        prog.add_multicast(BufferRef("sendbuf", 4, 4), BufferRef("recvbuf", 2, 4), 3, [1])
    assert e.value.code == "WriteWriteRace"
    prog.add_multicast(BufferRef("sendbuf", 4, 4), BufferRef("recvbuf", 4, 4), 3, [1])


def test_fence_rules():  # :95-110
    prog = base_program(4)
    with pytest.raises(HicclError) as e:
        prog.add_fence()
    assert e.value.code == "EmptyStep"
    prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1])
    prog.add_fence()
    with pytest.raises(HicclError):
        prog.add_fence()
    prog.add_multicast(BufferRef("recvbuf", 0, 4), BufferRef("recvbuf", 4, 4), 1, [2])
    assert len(steps_of(prog)) == 2
    prog.add_fence()
    assert "EmptyStep" in codes(prog.validate())


def test_write_write_race_via_append():  # :112-131 (the eager check fires)
    prog = CollectiveProgram(4)
    prog.declare_buffer("sendbuf", 8, input=True)
    prog.declare_buffer("recvbuf", 8)
    prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1])
    with pytest.raises(HicclError) as e:
        prog.add_multicast(BufferRef("sendbuf", 2, 4), BufferRef("recvbuf", 2, 4), 2, [1])
    assert e.value.code == "WriteWriteRace"


def test_read_write_overlap_within_a_step():  # :133-143
    prog = CollectiveProgram(4)
    prog.declare_buffer("sendbuf", 8, input=True)
    prog.declare_buffer("recvbuf", 8, input=True)
    prog.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1])
    prog.add_multicast(BufferRef("recvbuf", 0, 4), BufferRef("recvbuf", 4, 4), 1, [2])
    assert "ReadWriteRace" in codes(prog.validate())


def test_reads_of_never_written_non_input_ranges():  # :145-152
    prog = CollectiveProgram(4)
    prog.declare_buffer("sendbuf", 8, input=True)
    prog.declare_buffer("recvbuf", 8)
    prog.add_multicast(BufferRef("recvbuf", 0, 4), BufferRef("recvbuf", 4, 4), 0, [1])
    assert "UninitializedRead" in codes(prog.validate())


def test_empty_program_validates_clean():  # :154-157
    assert CollectiveProgram(4).validate() == []


def test_fig3_two_step_all_reduce_validates_clean():  # :159-179
    p, d = 3, 2
    prog = CollectiveProgram(p)
    prog.declare_buffer("sendbuf", p * d, input=True)
    prog.declare_buffer("recvbuf", p * d)
    for j in range(p):
        prog.add_reduction(BufferRef("sendbuf", j * d, d), BufferRef("recvbuf", j * d, d),
                           [0, 1, 2], j, ReduceOp.sum)
    prog.add_fence()
    for i in range(p):
        prog.add_multicast(BufferRef("recvbuf", i * d, d), BufferRef("recvbuf", i * d, d), i,
                           [r for r in range(p) if r != i])
    assert prog.validate() == []
    st = steps_of(prog)
    assert len(st) == 2
    m = st[1][0]
    assert m["send"] == m["recv"]  # in place


def test_serialization_round_trips_byte_identically():  # :181-191
    prog = base_program(4)
    prog.add_reduction(BufferRef("sendbuf", 0, 8), BufferRef("recvbuf", 0, 8), [0, 1, 2, 3], 2,
                       ReduceOp.max)
    prog.add_fence()
    prog.add_multicast(BufferRef("recvbuf", 0, 8), BufferRef("recvbuf", 8, 8), 2, [0, 1, 3])
    text = prog.serialize()
    back = CollectiveProgram.deserialize(text)
    assert back.serialize() == text
    assert back.id() == prog.id()


# ---- against the reference library itself --------------------------------

needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")


@needs_ref
def test_serialization_and_id_match_reference():
    ref = oracle.Reference()
    prog = base_program(4)
    prog.add_reduction(BufferRef("sendbuf", 0, 8), BufferRef("recvbuf", 0, 8), [3, 1, 0, 2, 1], 2,
                       ReduceOp.max)
    prog.add_fence()
    prog.add_multicast(BufferRef("recvbuf", 0, 8), BufferRef("recvbuf", 8, 8), 2, [0, 1, 3])
    text = prog.serialize()
    assert ref.roundtrip_program(text) == text


@needs_ref
def test_validate_codes_match_reference():
    ref = oracle.Reference()
    cases = []
    a = CollectiveProgram(4)
    a.declare_buffer("sendbuf", 8, input=True).declare_buffer("recvbuf", 8, input=True)
    a.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1])
    a.add_multicast(BufferRef("recvbuf", 0, 4), BufferRef("recvbuf", 4, 4), 1, [2])
    cases.append(a)
    b = CollectiveProgram(4)
    b.declare_buffer("sendbuf", 8, input=True).declare_buffer("recvbuf", 8)
    b.add_multicast(BufferRef("recvbuf", 0, 4), BufferRef("recvbuf", 4, 4), 0, [1])
    cases.append(b)
    c = base_program(4)
    c.add_multicast(BufferRef("sendbuf", 0, 4), BufferRef("recvbuf", 0, 4), 0, [1])
    c.add_fence()
    cases.append(c)
    for prog in cases:
        mine = [v.code for v in prog.validate()]
        assert mine == ref.validate_program(prog.serialize())
