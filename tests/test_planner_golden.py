"""Planner regression guard: the offline planner (tt_plan_offline, default
B200 description) must keep choosing the plans recorded in
tests/golden/planner_offline_plans.jsonl (written by
tools/plan_time/write_golden_plans.py; regenerated deliberately when a
planner rule changes -- the round-2 planner speed-ups were required to leave
every one of them unchanged).  This is a snapshot of the library's own
choices, not a parity reference: parity is the oracle's job."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools", "plan_time"))


def test_offline_plans_match_snapshot():
    import paper_1705_01598_b200 as tt
    from write_golden_plans import summary
    rows = [json.loads(l) for l in open(os.path.join(HERE, "golden", "planner_offline_plans.jsonl"))]
    assert len(rows) > 250
    bad = []
    for r in rows:
        got = json.loads(json.dumps(summary(tt.plan_offline(r["dims"], r["perm"], r["esize"])), sort_keys=True))
        if got != r["plan"]:
            bad.append((r["dims"], r["perm"], r["esize"]))
    assert not bad, f"{len(bad)} plans changed, first: {bad[:3]}"
