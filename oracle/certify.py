"""TEST INFRASTRUCTURE ONLY: the executed-timeline certificate of a DELTA step
on the GPU, shared by tests/ and __graft_entry__.smoke() so both apply the
same rule.

1. `DeltaRuntime.executed_timeline(findings)` runs one step with the
   executor's DEVICE-side action log (delta_rt_step_observed) and turns it into
   a reference Timeline; `findings` lists every disagreement between what the
   device ran and the lowered program (missing, duplicated, foreign or
   out-of-order actions).
2. The reference's own independent verifier, `oracle::replay_check`
   (/root/reference/proj/src/oracle.cpp:50-300, built unmodified into
   oracle/_ref), checks that timeline: budget never exceeded, no read of an
   absent tensor, no backward release, prefetch bursts within the limit,
   monotone non-overlapping streams (one compute stream, one copy stream).

Certified == no findings and no violations, unfiltered.  The default lowering
runs every copy on one copy stream in plan order (the reference's model), so
no finding class needs an exemption.
"""
from __future__ import annotations

from . import ref


def certify(rt) -> dict:
    """The budget checked is the CALLER's (rt.budget_bytes): the runtime may
    have planned under a smaller one so the packed arena fits it."""
    import dataclasses

    from paper_2203_15980_b200 import planner as P

    findings: list = []
    ev = rt.executed_timeline(findings)
    viol = None
    if ref.available():
        cfg = dataclasses.replace(rt.config, budget=getattr(rt, "budget_bytes", rt.config.budget))
        viol = ref.replay_check(rt.trace().to_json(), cfg, P.chrome_trace_events(ev))
    return {"findings": findings, "violations": viol, "events": ev,
            "ok": not findings and (viol is None or viol == [])}
