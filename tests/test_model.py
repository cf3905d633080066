"""Cost model and tuner (include/hiccl/model.hpp).

* the reference's closed forms at SPEC.md's spot values (acceptance 5, 7):
  Eq. (1) t_ring = 0.011748 s, Eq. (2) t_tree = 0.022115 s, Table-4 bounds;
* the B200 model against this round's committed measurements
  (profiles/r1/*.jsonl): within 10% at >= 64 MiB (20% for pipelined chains
  at >= 256 MiB);
* the tuner picks the compositions the measurements favour.
"""
import json
from pathlib import Path

import pytest

from paper_2408_05962_b200 import hiccl as H
from tests import harness

PROFILES = Path(__file__).resolve().parent.parent / "profiles" / "r1"


def test_eq1_eq2_spot_values():
    assert H.t_ring(1e-5, 2 ** 30, 4, 25e9, 32, 4) == pytest.approx(0.011748, rel=1e-4)
    assert H.t_tree(1e-5, 2 ** 30, 4, 25e9, 32, 4) == pytest.approx(0.022115, rel=1e-4)
    # alpha = 0, m -> large: ring independent of n, tree ~2x ring at n = 4
    r = H.t_ring(0, 2 ** 30, 4, 25e9, 4096, 4)
    t = H.t_tree(0, 2 ** 30, 4, 25e9, 4096, 4)
    assert t / r == pytest.approx(2.0, rel=1e-2)


def test_table4_bounds():
    kf = 4 * 25e9
    K = H.CollectiveKind
    assert H.bound(K.broadcast, 16, 4, 4, 25e9) == pytest.approx(kf)
    assert H.bound(K.all_gather, 16, 4, 4, 25e9) == pytest.approx(kf * 16 / 12)
    assert H.bound(K.all_reduce, 16, 4, 4, 25e9) == pytest.approx(66.7e9, rel=1e-3)
    assert H.bound(K.all_to_all, 16, 4, 4, 25e9) == pytest.approx(33.33e9, rel=1e-3)
    with pytest.raises(H.HicclError) as e:
        H.bound(K.all_reduce, 4, 4, 4, 25e9)
    assert e.value.code == "NoInterNodeBound"
    assert H.throughput(1e6, 8, 1e-3) == pytest.approx(8e9)


def measured():
    rows = []
    for f in ("sweep_p4.jsonl", "sweep_p4_chain.jsonl", "sweep_p2.jsonl"):
        path = PROFILES / f
        if path.exists():
            rows += [json.loads(l) for l in open(path)]
    return [r for r in rows if r.get("impl") == "hiccl" and r["bytes"] >= 64 << 20 and "us" in r]


KIND = {k.name: k.value for k in H.CollectiveKind}
FORM = {"single": 0, "multi": 1, "multi_alt": 2}


def test_model_matches_measurements():
    rows = measured()
    assert rows, "profiles/r1 measurements missing"
    checked = 0
    for r in rows:
        p = r["p"]
        kind = KIND[r["collective"]]
        form = FORM[r.get("formulation", "single")]
        d = r["bytes"] // (4 * p)
        g = r.get("g", p)
        plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, r.get("hierarchy", [p]), g,
                                       r.get("ring", 1), r.get("stripe", 1), r.get("pipeline", 1))
        pred = H.predict(plan, copy_mode=r.get("copy_mode", "push")) * 1e6
        if r.get("pipeline", 1) > 1:  # chains: per-slot cost of short tiles not modelled
            if r["bytes"] < 256 << 20:
                continue
            lo, hi = 0.8, 1.2
        else:
            lo, hi = 0.9, 1.1
        assert lo <= pred / r["us"] <= hi, (r["collective"], r["bytes"], p, pred, r["us"])
        checked += 1
    assert checked >= 20


def test_tuner_choices():
    K, F = H.CollectiveKind, H.Formulation
    ar_big = H.tune(K.all_reduce, 4, 1 << 26)
    assert ar_big["formulation"] == F.multi and ar_big["pipeline"] == 1
    assert H.tune(K.all_reduce, 4, 64)["formulation"] == F.single
    bc = H.tune(K.broadcast, 4, 1 << 26)
    assert bc["ring"] == 4 and bc["pipeline"] >= 16
    ag = H.tune(K.all_gather, 4, 1 << 26)
    assert ag["formulation"] == F.single and ag["pipeline"] == 1
    # small messages: tagged lines; large: point-to-point push
    assert H.tune(K.all_reduce, 4, 256)["copy_mode"] == "ll"
    assert H.tune(K.all_gather, 4, 1 << 16)["copy_mode"] == "ll"
    assert ar_big["copy_mode"] == "push"


def test_ll_model_matches_small_message_measurements():
    """Tagged-line timings (graph-replayed, p=4, profiles/r1/ll_graph_p4.jsonl,
    1 KiB - 64 MiB, all collectives and formulations) within a factor 1.5,
    most within 30%: the slot model has one line rate per direction and one
    for both directions busy, the hardware a continuum."""
    path = PROFILES / "ll_graph_p4.jsonl"
    rows = [json.loads(l) for l in open(path)] if path.exists() else []
    rows = [r for r in rows if r.get("impl") == "hiccl" and r.get("copy_mode") == "ll" and "us" in r]
    assert rows, "profiles/r1/ll_graph_p4.jsonl missing"
    close = 0
    for r in rows:
        p, kind = r["p"], KIND[r["collective"]]
        d = r["bytes"] // (4 * p)
        plan, _, _ = harness.make_plan(kind, FORM[r["formulation"]], p, d, 0, 0, [p], p, 1, 1, 1)
        pred = H.predict(plan, copy_mode="ll") * 1e6
        assert 0.65 <= pred / r["us"] <= 1.5, (r["collective"], r["bytes"], r["formulation"], pred, r["us"])
        close += 0.7 <= pred / r["us"] <= 1.3
    assert close >= 0.85 * len(rows)



def test_nvls_model_matches_measurements():
    # NVLS library (multimem) rows measured at p = 4 this round: fused
    # all-reduce, broadcast / reduce `single` lowered to one multimem
    # multicast / reduction (profiles/r1/nvls)
    rows = [json.loads(l) for f in ("rooted_and_ar_p4.jsonl", "reduce_forward_p4.jsonl")
            for l in (PROFILES / "nvls" / f).read_text().splitlines()]
    checked = 0
    for r in rows:
        if r["impl"] != "hiccl" or r["bytes"] < 64 << 20 or not r.get("nvls"):
            continue
        p = r["p"]
        plan, _, _ = harness.make_plan(KIND[r["collective"]], FORM[r["formulation"]], p,
                                       r["bytes"] // (4 * p))
        pred = H.predict_nvls(plan, "f32") * 1e6
        assert 0.9 <= pred / r["us"] <= 1.1, (r["collective"], r["bytes"], pred, r["us"])
        checked += 1
    assert checked >= 12


def test_nvls_tuner_choices():
    K = H.CollectiveKind
    gib = 1 << 30
    # all-reduce: the fused multimem path from p = 4 on (S(1+1/p) per link
    # direction against 2S(p-1)/p); point to point at p = 2
    assert not H.tune_nvls(K.all_reduce, 2, gib // 8, "f32")["nvls"]
    assert H.tune_nvls(K.all_reduce, 4, gib // 16, "f32")["nvls"]
    assert H.tune_nvls(K.all_reduce, 8, gib // 32, "f32")["nvls"]
    # no f32 max in the switch: the NVLS layout lowers nothing of the reduction
    plan, _, _ = harness.make_plan(7, 1, 4, gib // 16, op=1)
    assert H.predict_nvls(plan, "f32") > H.predict_nvls(harness.make_plan(7, 1, 4, gib // 16)[0], "f32")
    # broadcast of 16 MiB: one multimem.st from the root; all-gather stays p2p
    bc = H.tune_nvls(K.broadcast, 4, (16 << 20) // 16, "f32")
    assert bc["nvls"] and bc["formulation"] == H.Formulation.single
    assert not H.tune_nvls(K.all_gather, 4, gib // 16, "f32")["nvls"]
    # reduce of 64-256 MiB: reduce-scatter through the switch, each fold
    # forwarded to the root (fuse_forward_copy)
    rd = H.tune_nvls(K.reduce, 4, (256 << 20) // 16, "f32")
    assert rd["nvls"] and rd["formulation"] == H.Formulation.multi
