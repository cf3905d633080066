"""The command line (paper_2408_05962_b200/cli.py, mirroring the reference
CLI hiercoll_cli.cpp:184-361) and the persistent plan cache, on CPU."""
import json
from pathlib import Path

import pytest

from paper_2408_05962_b200 import cli
from paper_2408_05962_b200 import hiccl as H
from tests import harness

MACHINES = Path(cli.__file__).resolve().parent / "machines"
AR = ["--collective", "all_reduce", "--formulation", "multi"]


def run(capsys, *argv):
    rc = cli.main(list(argv))
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_plan_is_the_preset(capsys):
    rc, out, _ = run(capsys, "plan", *AR, "--p", "8", "--count", "16")
    assert rc == 0
    spec = H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, 16)
    assert out.rstrip("\n") == H.build(spec, 8).serialize().rstrip("\n")


def test_lower_pipeline_matrix(capsys, tmp_path):
    rc, out, _ = run(capsys, "lower", *AR, "--p", "8", "--count", "64", "--hierarchy", "2,4",
                     "--gpn", "4", "--stripe", "4", "--ring", "2")
    assert rc == 0 and json.loads(out)["format"] == "hiercoll-plan-v1"
    prog = tmp_path / "prog.json"
    run(capsys, "plan", *AR, "--p", "8", "--count", "64", "--out", str(prog))
    rc, out, _ = run(capsys, "pipeline", "--program", str(prog), "--p", "8",
                     "--machine", str(MACHINES / "b200x8_virtual_2x4.toy"), "--pipeline", "4")
    plan = json.loads(out)
    assert rc == 0 and plan["format"] == "hiercoll-pipelined-v1" and plan["slots"] >= 4
    # slot 0 of flat {4} AR multi: every rank sends d elements to every other
    rc, out, _ = run(capsys, "matrix", *AR, "--p", "4", "--count", "8", "--stage", "0")
    rows = [[int(x) for x in line.split(",")] for line in out.split()]
    assert rc == 0 and rows == [[32] * 4] * 4
    rc, _, err = run(capsys, "matrix", *AR, "--p", "4", "--count", "8", "--stage", "9")
    assert rc == 1 and "outside schedule" in err


def test_check_pass_and_rejected_ring(capsys):
    rc, out, _ = run(capsys, "check", *AR, "--p", "8", "--count", "100", "--hierarchy", "2,4",
                     "--gpn", "4", "--stripe", "4", "--ring", "2", "--pipeline", "4")
    assert rc == 0 and out.startswith("PASS")
    rc, out, _ = run(capsys, "check", "--collective", "all_gather", "--p", "8", "--count", "64",
                     "--machine", str(MACHINES / "b200x8_virtual_2x2x2.toy"), "--stripe", "2",
                     "--copy-mode", "ll")
    assert rc == 0 and out.startswith("PASS")
    # {8} g = 1 ring 2: the reference's block assembly would drop members
    # (SURVEY §0); rejected, exit 1 like the reference's errors
    rc, _, err = run(capsys, "check", *AR, "--p", "8", "--gpn", "1", "--ring", "2")
    assert rc == 1 and "InvalidConfig" in err


def test_usage_errors_exit_2(capsys):
    assert run(capsys, "bogus")[0] == 2
    assert run(capsys, "matrix", *AR)[0] == 2  # --stage required
    assert run(capsys, "plan", "--collective", "nope")[0] == 1


def test_simulate_sweep_tune(capsys):
    rc, out, _ = run(capsys, "simulate", *AR, "--p", "8", "--count", str(1 << 25))
    hdr, row = out.strip().split("\n")
    assert rc == 0 and hdr.startswith("collective,")
    t_p2p = float(row.split(",")[8])
    rc, out, _ = run(capsys, "simulate", *AR, "--p", "8", "--count", str(1 << 25), "--nvls")
    t_nvls = float(out.strip().split("\n")[1].split(",")[8])
    assert t_nvls < t_p2p
    plan, _, _ = harness.make_plan(7, 1, 8, 1 << 25)
    assert t_p2p == pytest.approx(H.predict(plan), rel=1e-6)
    rc, out, _ = run(capsys, "sweep", "--collective", "broadcast", "--p", "4", "--counts",
                     "1024,65536", "--ring", "1,4", "--gpn", "1", "--pipeline", "1,8")
    assert rc == 0 and len(out.strip().split("\n")) == 1 + 2 * 2 * 2
    rc, out, _ = run(capsys, "tune", "--collective", "all_reduce", "--p", "8", "--count",
                     str(1 << 22), "--nvls")
    t = json.loads(out)
    assert rc == 0 and t["nvls"] and t["formulation"] == "multi"


def test_bounds_spot_value(capsys):
    # SPEC.md acceptance: AR bound at p=16, g=4, k=4, f=25 GB/s is 66.7 GB/s
    rc, out, _ = run(capsys, "bounds", "--p", "16", "--gpn", "4", "--nics", "4",
                     "--nic-bandwidth", "25e9")
    rows = {l.split(",")[0]: l.split(",") for l in out.strip().split("\n")[1:]}
    assert rc == 0 and float(rows["all_reduce"][6]) == pytest.approx(66.6667, rel=1e-4)
    assert float(rows["all_to_all"][6]) == pytest.approx(33.3333, rel=1e-4)


def test_plan_cache(tmp_path):
    spec = H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, 999)
    prog = H.build(spec, 8)
    machine = H.Machine([2, 4], 4)
    cache = H.PlanCache(str(tmp_path))
    a = cache.lower(prog, machine, ring=2, stripe=4, pipeline=3)
    assert (cache.hits, cache.misses) == (0, 1)
    b = H.PlanCache(str(tmp_path)).lower(prog, machine, ring=2, stripe=4, pipeline=3)
    assert a.serialize() == b.serialize()
    assert b.serialize() == H.lower(prog, machine, ring=2, stripe=4, pipeline=3).serialize()
    c = cache.lower(prog, machine, ring=2, stripe=4, pipeline=4)  # another key
    assert cache.misses == 2 and c.slots != a.slots
    assert len(list(tmp_path.glob("*.json"))) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("coll,form", [("all_reduce", "multi"), ("all_to_all", "single"),
                                       ("broadcast", "single"), ("reduce_scatter", "single")])
def test_check_runs_on_the_device(capsys, coll, form):
    rc, out, _ = run(capsys, "check", "--collective", coll, "--formulation", form, "--p", "4",
                     "--count", "1000", "--gpus", "1")
    assert rc == 0 and "device run" in out, out
