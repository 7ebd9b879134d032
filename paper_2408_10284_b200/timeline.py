"""Physical timeline of a decode session (moe_decode_timeline_write): reader and validators.

The JSONL follows the reference's timeline schema (inc/io.hpp:402-417: stream, kind, start, end,
expert, token, layer, tile) with CUDA-event times in microseconds, plus physical fields:
  tile_transfer (stream "comm"):  request ("on_demand" | "prefetch"), promoted, evicts, job
  expert_compute / tile_compute:  launch (FFN launch id), fill (copy job whose tiles filled the slot;
                                  -1 = initial residency)
  wait (stream "compute"):        the compute stream blocked on tile `tile` of copy job `job`
  gate:                           a router (K1) launch
The validators restate the reference's own (proj/tests/support/timeline_checks.hpp:24-55) on real
timestamps: causality (no segment computes before the copy of the bytes it reads has landed),
stream exclusivity (one copy stream, one compute stream: no overlap; the segments of one FFN launch
share its interval), and counting identities against the session's metrics and counters.
"""
from __future__ import annotations

import json
from collections import defaultdict


def load(path) -> list[dict]:
    with open(path) as f:
        return [json.loads(line) for line in f if line.strip()]


def check_causality(events: list[dict], slack_us: float = 0.0) -> list[str]:
    """Every FFN segment whose slot was filled by a copy job starts after that job's copy of the
    same tile ended (inc/simulator.hpp semantics: compute after transfer completion).  A recording
    that starts mid-session cannot see copies that began before it: segments reading a job whose
    tile 0 is not in the timeline are not checked."""
    ends = {}
    for e in events:
        if e["kind"] == "tile_transfer":
            ends[(e["job"], e["tile"])] = e["end"]
    in_window = {job for job, tile in ends if tile == 0}
    problems = []
    for e in events:
        if e["kind"] in ("expert_compute", "tile_compute") and e["fill"] in in_window:
            end = ends.get((e["fill"], e["tile"]))
            if end is None:
                problems.append(f"launch {e['launch']}: layer {e['layer']} expert {e['expert']} tile {e['tile']} reads "
                                f"copy job {e['fill']} whose tile was never transferred")
            elif end > e["start"] + slack_us:
                problems.append(f"launch {e['launch']}: layer {e['layer']} expert {e['expert']} tile {e['tile']} starts "
                                f"at {e['start']:.3f} us before its copy ended at {end:.3f} us")
    return problems


def check_stream_exclusivity(events: list[dict], slack_us: float = 0.0) -> list[str]:
    """Intervals on one stream never overlap (an FFN launch's segments count as one interval)."""
    problems = []
    per_stream = defaultdict(dict)
    for e in events:
        key = ("launch", e["launch"]) if "launch" in e else ("event", id(e))
        per_stream[e["stream"]].setdefault(key, (e["start"], e["end"], e["kind"]))
    for stream, ivs in per_stream.items():
        seq = sorted(ivs.values())
        for (s0, e0, k0), (s1, e1, k1) in zip(seq, seq[1:]):
            if e0 > s1 + slack_us:
                problems.append(f"overlap on {stream}: {k0} [{s0:.3f}, {e0:.3f}] and {k1} [{s1:.3f}, {e1:.3f}]")
    return problems


def check_conservation(events: list[dict], metrics: dict, stats: dict | None = None) -> list[str]:
    """Counting identities: every activated (token, layer, expert) computed exactly once, the
    non-resident ones are the on-demand loads, and every tile copy appears once."""
    problems = []
    computed = {}
    for e in events:
        if e["kind"] in ("expert_compute", "tile_compute"):
            key = (e["token"], e["layer"], e["expert"])
            computed.setdefault(key, set()).add(e["kind"])
    on_demand = sum(1 for k in computed.values() if "tile_compute" in k)
    if len(computed) != metrics["experts_activated_total"]:
        problems.append(f"activations: timeline {len(computed)} vs metrics {metrics['experts_activated_total']}")
    if on_demand != metrics["on_demand_loads"]:
        problems.append(f"on-demand computes: timeline {on_demand} vs metrics {metrics['on_demand_loads']}")
    if stats is not None:
        copies = sum(1 for e in events if e["kind"] == "tile_transfer")
        if copies != stats["tile_copies"]:
            problems.append(f"tile copies: timeline {copies} vs counters {stats['tile_copies']}")
    return problems
