"""Executed budget x policy x heuristic comparison grid.

The reference's `run_comparison` (src/engine.cpp:646-671) plans every
(budget, policy, heuristic) cell and `comparison_to_csv`
(src/metrics.cpp:314-328) renders one Report row per cell against the
unconstrained baseline.  Here every cell is EXECUTED on the B200 by the DELTA
runtime: planned by libdelta (the same decisions as the reference, see
`planner.comparison`), lowered onto the HBM arena, captured as a CUDA graph
and timed; the row keeps the reference's CSV header with the measured
quantities in place of the simulated ones:

  peak_bytes            the arena footprint the step really used
  baseline_peak_bytes   the no-eviction arena footprint
  wall_time_us          measured µs per training step (CUDA events)
  baseline_wall_time_us measured µs per no-eviction step
  saving / overhead     recomputed from those
  counts, stall, overlap as planned (the plan the GPU executed)

`detail` rows add the simulated wall time, whether the step was bit-identical
to the no-eviction step (loss and every gradient), and the plan's budget when
the arena refit (DeltaRuntime.plan) planned under a smaller one.
"""
from __future__ import annotations

import csv
import io

import torch

from . import planner as P

CSV_HEADER = ("trace,budget,policy,heuristic,peak_bytes,baseline_peak_bytes,saving_fraction,"
              "wall_time_us,baseline_wall_time_us,overhead_fraction,evict,offload,reload,"
              "recompute,prefetch_reload,total_stall_us,overlap_ratio,infeasible")


def _g(x: float) -> str:
    """std::ostream's default formatting of a double (6 significant digits)"""
    return format(x, ".6g")


def _timed(rt, warmup: int, steps: int) -> float:
    rt.capture()
    for _ in range(warmup):
        rt.step_device()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(rt.stream)
    for _ in range(steps):
        rt.step_device()
    e1.record(rt.stream)
    torch.cuda.synchronize()
    rt.graph = rt.graphs = None
    return e0.elapsed_time(e1) / steps * 1e3  # µs


def _one_step(rt):
    with torch.cuda.stream(rt.stream):
        rt.run_program()
    torch.cuda.synchronize()
    return rt.loss.clone(), rt.params.grad.clone()


def executed_comparison(rt, budget_fractions, policies, heuristics, steps: int = 5,
                        warmup: int = 2):
    """Run the grid on `rt` (inputs already in its device slots; lr is held
    at 0 so every cell steps on the same weights).  Returns (csv_text,
    detail_rows)."""
    lr = rt.lr
    rt.lr = 0.0
    try:
        rt.plan(None)
        base_prog = rt.program
        base_us = _timed(rt, warmup, steps)
        loss0, grad0 = _one_step(rt)
        base_peak = rt.baseline_peak()
        trace = rt.trace()
        name = trace.name
        rows, detail = [], []
        for f in budget_fractions:
            budget = int(base_peak * f)
            for pol in policies:
                for h in heuristics:
                    cell = {"budget_fraction": f, "budget": budget, "policy": pol.name,
                            "heuristic": h.name}
                    try:
                        prog = rt.plan(budget=budget, policy=pol, heuristic=h)
                    except RuntimeError as e:
                        # not executed.  Infeasible in the plan: the reference's
                        # row as is.  Feasible in the plan but its arena cannot
                        # be packed within the budget (fragmentation, see
                        # DeltaRuntime.plan): the planned row marked infeasible,
                        # with no measured time
                        cfg = rt.engine_config(budget, pol, heuristic=h)
                        ref = next(csv.DictReader(io.StringIO(
                            P.comparison(trace, [budget], [pol], [h], cfg))))
                        planned_ok = ref["infeasible"] == "false"
                        if planned_ok:
                            ref.update(wall_time_us="0", baseline_wall_time_us=str(int(round(base_us))),
                                       overhead_fraction="0", infeasible="true")
                        rows.append(",".join(ref[k] for k in CSV_HEADER.split(",")))
                        cell.update(infeasible=True, error=str(e)[:160],
                                    reason=("arena packing exceeds the budget (fragmentation)"
                                            if planned_ok else "plan infeasible"))
                        detail.append(cell)
                        continue
                    cfg = rt.config
                    planned = next(csv.DictReader(io.StringIO(
                        P.comparison(trace, [cfg.budget], [pol], [h], cfg))))
                    us = _timed(rt, warmup, steps)
                    loss, grad = _one_step(rt)
                    bit = bool(torch.equal(loss, loss0) and torch.equal(grad, grad0))
                    saving = 1.0 - prog.arena_bytes / base_prog.arena_bytes
                    overhead = us / base_us - 1.0
                    rows.append(",".join([
                        name, str(budget), planned["policy"], planned["heuristic"],
                        str(prog.arena_bytes), str(base_prog.arena_bytes), _g(saving),
                        str(int(round(us))), str(int(round(base_us))), _g(overhead),
                        planned["evict"], planned["offload"], planned["reload"],
                        planned["recompute"], planned["prefetch_reload"],
                        planned["total_stall_us"], planned["overlap_ratio"], "false"]))
                    cell.update(infeasible=False, arena_bytes=prog.arena_bytes,
                                planned_budget=cfg.budget, measured_us=round(us, 1),
                                baseline_us=round(base_us, 1),
                                simulated_wall_us=int(planned["wall_time_us"]),
                                simulated_baseline_us=int(planned["baseline_wall_time_us"]),
                                images_per_s=round(rt.batch / (us * 1e-6), 1),
                                no_eviction_ratio=round(base_us / us, 4),
                                bit_identical=bit)
                    detail.append(cell)
        return CSV_HEADER + "\n" + "\n".join(rows) + "\n", detail
    finally:
        rt.lr = lr
