"""CPU: the physical-timeline validators (paper_2408_10284_b200/timeline.py, restating
proj/tests/support/timeline_checks.hpp:24-55) accept a consistent timeline and flag each violation."""
from paper_2408_10284_b200 import timeline as TL


def _tr(job, tile, s, e, layer=0, expert=1, req="on_demand"):
    return {"stream": "comm", "kind": "tile_transfer", "start": s, "end": e, "expert": expert, "token": 0,
            "layer": layer, "tile": tile, "request": req, "promoted": False, "evicts": -1, "job": job}


def _cp(launch, tile, s, e, fill, expert=1, kind="tile_compute", token=0, layer=0):
    return {"stream": "compute", "kind": kind, "start": s, "end": e, "expert": expert, "token": token, "layer": layer,
            "tile": tile, "launch": launch, "fill": fill}


GOOD = [_tr(0, 0, 0.0, 10.0), _tr(0, 1, 10.0, 20.0),
        {"stream": "compute", "kind": "wait", "start": 1.0, "end": 20.5, "expert": 1, "token": 0, "layer": 0,
         "tile": 1, "job": 0},
        _cp(0, 0, 21.0, 30.0, 0), _cp(0, 1, 21.0, 30.0, 0),
        _cp(1, 0, 31.0, 40.0, -1, expert=2, kind="expert_compute"), _cp(1, 1, 31.0, 40.0, -1, expert=2, kind="expert_compute")]
METRICS = {"experts_activated_total": 2, "on_demand_loads": 1}


def test_consistent_timeline_passes():
    assert TL.check_causality(GOOD) == []
    assert TL.check_stream_exclusivity(GOOD) == []
    assert TL.check_conservation(GOOD, METRICS, {"tile_copies": 2}) == []


def test_compute_before_copy_is_flagged():
    bad = GOOD[:3] + [_cp(0, 0, 15.0, 30.0, 0), _cp(0, 1, 15.0, 30.0, 0)] + GOOD[5:]
    probs = TL.check_causality(bad)
    assert len(probs) == 1 and "tile 1" in probs[0]
    assert TL.check_causality(GOOD[:3] + [_cp(0, 3, 21.0, 30.0, 0)])  # tile never copied
    # a job that started before the recording (tile 0 absent) is not checked
    assert TL.check_causality(GOOD + [_cp(3, 0, 50.0, 60.0, 9)]) == []


def test_overlaps_are_flagged():
    assert TL.check_stream_exclusivity(GOOD + [_tr(1, 0, 19.0, 25.0)])
    assert TL.check_stream_exclusivity(GOOD + [_cp(2, 0, 35.0, 45.0, -1)])
    # the segments of one launch share an interval: not an overlap
    assert TL.check_stream_exclusivity(GOOD + [_cp(1, 2, 31.0, 40.0, -1, expert=2, kind="expert_compute")]) == []


def test_counting_identities_are_checked():
    assert TL.check_conservation(GOOD, {"experts_activated_total": 3, "on_demand_loads": 1})
    assert TL.check_conservation(GOOD, {"experts_activated_total": 2, "on_demand_loads": 0})
    assert TL.check_conservation(GOOD, METRICS, {"tile_copies": 3})
