#!/usr/bin/env python
"""bench: ResNet-50 training images/s on B200 under a 50% DELTA activation budget.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full training step (forward, backward, SGD update) of
ResNet-50 at batch 256/GPU (224x224, bf16 activations, synthetic ImageNet-shaped
data, random init) executed by the DELTA runtime under an activation-memory
budget of 50% of the no-eviction peak.  Inputs: the ~5 GB activation working
set per step exceeds the 126 MB L2 (no flush needed).  Prints ONE JSON line
(rank 0).  Multi-GPU: launched by torchrun, one DELTA instance per GPU
(identical plans: cost tables max-reduced across ranks), NCCL gradient
all-reduce; time = max over ranks.

--impl reference times the reference's own CPU implementation of the DELTA
path (the unmodified C++ simulator, oracle/_ref, run_iteration on the same
ResNet-50 trace) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

PCIE5_X16_GBS = 64.0  # nominal per direction (32 GT/s x 16 lanes, 128b/130b)
METRIC = "ResNet-50 imgs/sec at 50% activation budget; peak act GB; max batch vs baseline"
TRACE_FIXTURE = os.path.join(HERE, "tests", "golden", "resnet50_bs256_trace.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--depth", type=int, default=50)
    ap.add_argument("--budget", type=float, default=0.5)
    ap.add_argument("--anchors", default="out+narrow")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=10.0)
    ap.add_argument("--export-trace", default="")
    ap.add_argument("--detail", default="", help="where to write the full JSON record")
    ap.add_argument("--bert-batch", type=int, default=32,
                    help="config 5 (BERT-large seq 512) batch per GPU; 0 skips the BERT section")
    ap.add_argument("--bert-budget", type=float, default=0.4)
    ap.add_argument("--bert-steps", type=int, default=10)
    ap.add_argument("--no-verify-max-batch", action="store_true",
                    help="skip the real training steps at the planner-decided max batches")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(device_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- config 5
def bert_section(args, world, rank, dp, barrier, max_over_ranks):
    """Config 5: BERT-large (24 x 1024, 16 heads, FFN 4096, seq 512, SQuAD span
    head, AdamW, dropout 0.1) under a DELTA activation budget on this GPU (one
    DELTA instance per rank, NCCL gradient all-reduce).  Same protocol as the
    headline: parity gate (DELTA step == no-eviction step bit for bit),
    graph-replayed steps timed with CUDA events (max over ranks), end to end
    through BertRuntime.train with pinned host batches."""
    import torch
    from paper_2203_15980_b200 import bert as BT
    cfg = BT.BertConfig(batch=args.bert_batch)
    rt = BT.BertRuntime(cfg, seed=0)
    rt.dp = dp
    batches = [rt.synthetic_batch(1000 * rank + i) for i in range(2)]
    for slot in range(2):
        for d, h in zip(rt.in_slots[slot], batches[0]):
            d.copy_(h)
    rt.measure_costs(iters=3)
    if dp is not None:
        from paper_2203_15980_b200.runtime import agree_cost_table
        rt.link_gbs = agree_cost_table(rt.g, rt.link_gbs, dp, device="cuda")
    lr = rt.lr
    rt.lr = 0.0
    rng0 = rt.rng.clone()
    rt.plan(None)
    rt.step_device()
    loss_ref, grad_ref = rt.loss.clone(), rt.params.grad.clone()
    rt.rng.copy_(rng0)
    prog = rt.plan(args.bert_budget)
    rt.step_device()
    torch.cuda.synchronize()
    parity = {"loss_equal": bool(torch.equal(loss_ref, rt.loss)),
              "grads_equal": bool(torch.equal(grad_ref, rt.params.grad)),
              "loss": round(float(loss_ref.item()), 6)}
    del grad_ref
    rt.lr = lr
    if not (parity["loss_equal"] and parity["grads_equal"]):
        raise SystemExit(f"BERT parity gate failed: DELTA step != no-eviction step {parity}")
    n = args.bert_steps

    def timed(frac):
        p = rt.plan(frac)
        rt.step_device()
        rt.capture()
        for _ in range(max(3, args.warmup)):
            rt.step_device()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(rt.stream)
        for _ in range(n):
            rt.step_device()
        e1.record(rt.stream)
        torch.cuda.synchronize()
        barrier()
        return p, max_over_ranks(e0.elapsed_time(e1) / n)

    bp, base_ms = timed(None)
    dprog, ms = timed(args.bert_budget)
    launches = rt.executor.launches_per_step
    rt.train([batches[i % 2] for i in range(3)])
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    losses = rt.train([batches[i % 2] for i in range(n)])
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / n)
    flops = sum(nd.flops for nd in rt.nodes)  # first productions (recomputes extra)
    B, S = cfg.batch, cfg.seq
    # the reference simulator planning this run's BERT trace on one host core
    cpu = None
    if rank == 0:
        try:
            from oracle import ref as oref
            if oref.available():
                tj = rt.trace().to_json()
                ns = oref.time_run_ns(tj, rt.config, 50)
                sim = oref.run(tj, rt.config)
                cpu = {"value": round(B / (sim["wall_time_us"] * 1e-6), 1), "unit": "seq/s",
                       "cores": 1, "kind": "reference",
                       "sample": f"reference simulator on this run's {len(rt.nodes)}-node BERT trace: "
                                 f"predicted step {sim['wall_time_us']} us (simulated, not trained); "
                                 f"{ns * 1e-3:.0f} us per run_iteration on one core",
                       "same_decisions": sim["decisions"] == [[n, int(a)] for n, a in dprog.decisions]}
        except Exception as e:  # noqa: BLE001 - never breaks the bench
            cpu = {"value": None, "sample": f"unavailable: {e}"}
    out = {
        "workload": f"BERT-large (24x1024, 16 heads, FFN 4096) seq {S}, batch {B}/GPU, SQuAD span "
                    f"head, AdamW, dropout 0.1, DELTA at {int(args.bert_budget * 100)}% activation "
                    "budget (config 5)",
        "seq_per_s": round(world * B / (ms * 1e-3), 1),
        "tokens_per_s": round(world * B * S / (ms * 1e-3), 0),
        "ms_per_step": round(ms, 3),
        "no_eviction_seq_per_s": round(world * B / (base_ms * 1e-3), 1),
        "no_eviction_ratio": round(base_ms / ms, 4),
        "peak_act_gb": round(dprog.arena_bytes / 1e9, 3),
        "peak_act_gb_no_eviction": round(bp.arena_bytes / 1e9, 3),
        "plan": dprog.plan_counts,
        "parity": parity,
        "model_tflops": round(flops / (ms * 1e-3) / 1e12, 1),
        "e2e": {"seq_per_s": round(world * B / e2e_s, 1),
                "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in batches[0]),
                "d2h_bytes_per_step": 4,
                "loss_first_last": [round(losses[0], 4), round(losses[-1], 4)]},
        "gpu_launches": launches * n,
        "cpu_baseline": cpu,
        "data": "synthetic token ids / segments / span labels, random init (no checkpoint)",
    }
    del rt
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------- config 3
def verify_batch(depth, batch, anchors, delta, per_sample, link_gbs, cap, MB):
    """One ResNet training step (plus a timed second one) at `batch` under the
    DELTA plan whose budget is the HBM the planner search gave it (or no
    eviction): the planner's max-batch answer, trained for real."""
    import torch
    from paper_2203_15980_b200.runtime import DeltaRuntime
    torch.cuda.reset_peak_memory_stats()
    rt = DeltaRuntime(depth, batch, seed=0, anchors=anchors)
    ps = MB.per_sample_costs(depth, per_sample)
    for n in rt.nodes:
        n.cost_us = max(1, int(round(ps.get(n.name, 1 / 256) * batch)))
    rt.link_gbs = link_gbs
    room = cap - MB.workspace_bytes(rt.g, batch)
    prog = rt.plan(budget=room) if delta else rt.plan(None)
    gen = torch.Generator().manual_seed(7)
    x = torch.zeros(rt.x_dev.shape, dtype=torch.bfloat16)
    k = min(batch, 256)  # random images in the first 256 slots (host memory stays modest)
    x[:k, ..., :3] = torch.randn(k, 224, 224, 3, generator=gen).to(torch.bfloat16)
    y = torch.randint(0, 1000, (batch,), generator=gen)
    rt.step(x, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loss = rt.step(x, y)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out = {"batch": batch, "anchors": anchors, "arena_gb": round(prog.arena_bytes / 1e9, 2),
           "plan": prog.plan_counts, "peak_alloc_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2),
           "img_s": round(batch / dt, 1), "loss": round(loss, 4)}
    del rt, prog
    return out


# -------------------------------------------------------- reference arm
_PLAN_WORKER = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from oracle import ref
tj = open(sys.argv[2]).read()
m = json.load(open(sys.argv[3]))
cfg = ref.config(m["budget"], tuple(m["bandwidth_bytes_per_us"]), (1, 1))
one = ref.time_run_ns(tj, cfg, 3)
iters = max(1, int(float(sys.argv[4]) * 1e9 / one))
print(ref.time_run_ns(tj, cfg, iters), iters)
"""


def host_cpu():
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    try:
        nproc = int(subprocess.run(["nproc"], capture_output=True, text=True, timeout=10).stdout)
    except Exception:  # noqa: BLE001
        nproc = os.cpu_count() or 1
    return nproc, model


def pinned_planners(trace_path, meta_path, seconds):
    """One single-threaded reference planner process per host core, each
    pinned to its own core with taskset; returns
    (plans/s summed over processes, per-process ns/plan)."""
    nproc, _ = host_cpu()
    procs = []
    for c in range(nproc):
        cmd = [sys.executable, "-c", _PLAN_WORKER, HERE, trace_path, meta_path, str(seconds)]
        if shutil.which("taskset"):
            cmd = ["taskset", "-c", str(c)] + cmd
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True))
    ns = []
    for p in procs:
        out, _ = p.communicate(timeout=600)
        ns.append(float(out.split()[0]))
    return sum(1e9 / v for v in ns), ns


def reference_arm(args, rank):
    """The reference's own CPU implementation of the DELTA path: the
    unmodified C++ simulator (oracle/_ref, built from /root/reference/proj/src)
    planning the ResNet-50 bs256 step at the 50% budget.  No product code is
    imported here.  Its answer to the headline metric is the step time it
    PREDICTS for that plan (`value` = batch / simulated wall time, the
    reference's model of a training step — labelled as simulated); the CPU
    cost of producing it is `planning` (µs per plan on one core, and plans/s
    with one pinned single-threaded planner per host core)."""
    if rank != 0:
        return
    from oracle import ref as oref
    if not oref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    trace_json = open(TRACE_FIXTURE).read()
    meta_path = TRACE_FIXTURE.replace(".json", ".meta.json")
    meta = json.load(open(meta_path))
    cfg = oref.config(meta["budget"], tuple(meta["bandwidth_bytes_per_us"]), (1, 1))
    B = meta["batch"]
    # warm-up + timed steps: one step = the reference planning this training
    # step once (run_iteration, one host thread)
    for _ in range(args.warmup):
        oref.time_run_ns(trace_json, cfg, 1)
    step_ns = [oref.time_run_ns(trace_json, cfg, 1) for _ in range(args.steps)]
    out = oref.run(trace_json, cfg)
    sim_us = out["wall_time_us"]
    value = B / (sim_us * 1e-6)
    plans_s, per_proc = pinned_planners(TRACE_FIXTURE, meta_path, min(3.0, args.cpu_sample_s))
    nproc, model = host_cpu()
    us_plan = statistics.median(step_ns) * 1e-3
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sim_us * 1e-3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "value_kind": "simulated: batch / the reference simulator's predicted step time for "
                      "its own DELTA plan of this step (its model of training, not a training run)",
        "config": {"workload": f"ResNet-50 training step, batch {B}/GPU, DELTA at "
                               f"{int(args.budget * 100)}% activation budget (reference simulator "
                               "run_iteration on the B200-measured trace, tests/golden)",
                   "global_batch": B, "budget_bytes": meta["budget"],
                   "trace": os.path.relpath(TRACE_FIXTURE, HERE)},
        "planning": {"us_per_plan_1core": round(us_plan, 1),
                     "pinned_processes": nproc, "plans_per_s_all_cores": round(plans_s, 1),
                     "cpu": model, "nproc": nproc,
                     "us_per_plan_per_process": [round(v * 1e-3, 1) for v in per_proc]},
        "cpu_baseline": {"value": round(value, 1), "unit": "images/s", "cores": 1,
                         "kind": "reference",
                         "sample": f"{args.steps} x run_iteration of the "
                                   f"{len(json.loads(trace_json)['nodes'])}-node ResNet-50 bs{B} "
                                   f"trace, one thread ({us_plan:.0f} us/plan); {nproc} pinned "
                                   f"planner processes: {plans_s:.0f} plans/s"},
        "e2e": {"value": round(value, 1), "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "simulated": {"wall_time_us": sim_us, "decisions": len(out["decisions"]),
                      "stall_us": out.get("total_stall_us")},
    }))


# ------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2203_15980_b200 import kernels as K
    from paper_2203_15980_b200 import planner as P
    from paper_2203_15980_b200.runtime import DeltaRuntime

    torch.cuda.set_device(local)
    dp = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dp = dist.group.WORLD

    def barrier():
        if dp is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dp is None:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    B = args.batch
    free_hbm = torch.cuda.mem_get_info()[0]
    rt = DeltaRuntime(args.depth, B, seed=0, anchors=args.anchors)
    rt.dp = dp

    gen = torch.Generator().manual_seed(1234 + rank)
    xs = []
    for i in range(2):
        x = torch.zeros(rt.x_dev.shape, dtype=torch.bfloat16).pin_memory()
        x[..., :3] = torch.randn(B, 224, 224, 3, generator=gen).to(torch.bfloat16)
        y = torch.randint(0, 1000, (B,), generator=gen).pin_memory()
        xs.append((x, y))
    for slot in range(2):
        rt.x_slots[slot].copy_(xs[0][0])
        rt.y_slots[slot].copy_(xs[0][1])

    # ---- GPU cost model on representative inputs (identical on every rank:
    # ---- max over ranks) ----
    rt.measure_costs(iters=3)
    if dp is not None:
        from paper_2203_15980_b200.runtime import agree_cost_table
        rt.link_gbs = agree_cost_table(rt.g, rt.link_gbs, dp, device="cuda")

    # ---- parity gate at THIS configuration, before anything is timed: one
    # ---- eager no-eviction step and one eager DELTA step on the same batch
    # ---- (lr 0) must agree bit for bit — loss and every gradient ----
    lr = rt.lr
    rt.lr = 0.0
    rt.plan(None)
    rt.step_device()
    loss_ref = rt.loss.clone()
    grad_ref = rt.params.grad.clone()
    rt.plan(args.budget)
    rt.step_device()
    torch.cuda.synchronize()
    parity = {"loss_equal": bool(torch.equal(loss_ref, rt.loss)),
              "grads_equal": bool(torch.equal(grad_ref, rt.params.grad)),
              "loss": round(float(loss_ref.item()), 6)}
    del grad_ref
    rt.lr = lr
    if not (parity["loss_equal"] and parity["grads_equal"]):
        raise SystemExit(f"parity gate failed at batch {B}: DELTA step != no-eviction step {parity}")

    def timed_device_steps(n_warm, n_steps):
        for _ in range(n_warm):
            rt.step_device()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(rt.stream)
        for _ in range(n_steps):
            rt.step_device()
        e1.record(rt.stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / n_steps)

    graph_state = {"captured": not args.no_graph}

    def prepare(budget_fraction):
        prog = rt.plan(budget_fraction)
        rt.step_device()  # eager warm step (allocator, first-launch attributes)
        torch.cuda.synchronize()
        if not args.no_graph:
            try:
                rt.capture()
            except Exception as e:  # noqa: BLE001 - e.g. a collective not capturable here
                if dp is None:
                    raise
                # reported in the JSON line (config.graph), never silent
                graph_state["captured"] = False
                graph_state["error"] = str(e)[:200]
                print(json.dumps({"warning": f"CUDA graph capture with NCCL failed ({e}); "
                                             "running eager steps"}), file=sys.stderr)
                rt.graph = rt.graphs = None
                torch.cuda.synchronize()
        # our kernel launches per step, counted from the bound recipes
        return prog, rt.executor.launches_per_step

    # ---- no-eviction upper bound (same kernels, Baseline policy) ----
    base_prog, _ = prepare(None)
    base_ms = timed_device_steps(args.warmup, args.steps)
    base_arena = base_prog.arena_bytes
    base_peak = base_prog.pool_peak_bytes

    # ---- DELTA at the budget ----
    prog, launches = prepare(args.budget)
    trace = rt.trace()
    if args.export_trace and rank == 0:
        with open(args.export_trace, "w") as f:
            f.write(trace.to_json())
        with open(args.export_trace.replace(".json", ".meta.json"), "w") as f:
            json.dump({"batch": B, "budget": rt.config.budget,
                       "bandwidth_bytes_per_us": list(rt.config.cost_model.bandwidth_bytes_per_us),
                       "anchors": args.anchors, "depth": args.depth}, f)
    clocks = ClockSampler(local)
    delta_ms = timed_device_steps(args.warmup, args.steps)
    clk = clocks.stop()

    # ---- end to end through the public API: host batches -> steps -> losses
    # ---- (DeltaRuntime.train: H2D of every batch overlapped with the
    # ---- previous step on a copy-engine stream, D2H of every loss) ----
    rt.train([xs[i % 2] for i in range(args.warmup)])
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    losses = rt.train([xs[i % 2] for i in range(args.steps)])
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    h2d_bytes = xs[0][0].numel() * 2 + xs[0][1].numel() * 8
    d2h_bytes = 4

    # ---- roofline of the dominant hand-written kernel (conv_fwd, tcgen05) ----
    saved_graph = rt.graph
    rt.graph = None
    for _ in range(2):  # the second eager pass is the one timed
        timing = {}
        with torch.cuda.stream(rt.stream):
            rt.run_program(timing=timing)
        torch.cuda.synchronize()
    rt.graph = saved_graph
    hbm_peak, tc_peak, tc_sus, peak_kind = measured_peaks()
    # DRAM bytes per forward conv launch from the committed ncu capture
    # (scripts/gpu_traffic.sh + scripts/conv_traffic.py), vs its algorithmic bytes
    conv_traffic = {}
    try:
        with open(os.path.join(HERE, "profiles", "r01_conv_traffic.json")) as f:
            t = json.load(f)
        conv_traffic = {"dram_bytes_per_launch": t["dram_bytes_per_launch"],
                        "note": f"ncu dram read+write per forward conv launch = "
                                f"{t['traffic_over_algorithmic']}x its algorithmic bytes "
                                f"({t['launches']} launches, profiles/r01_conv_traffic.json)"}
    except Exception:  # noqa: BLE001
        conv_traffic = {}
    conv_ms, conv_flops, conv_n, all_ms, conv_roof_ms = 0.0, 0.0, 0, 0.0, 0.0
    kinds = {}
    rc = {"launches": 0, "ms": 0.0, "roofline_ms": 0.0, "flops": 0.0, "bytes": 0.0, "by_op": {}}
    swap_ms, swap_bytes, swap_n = 0.0, 0, 0
    # the whole step against its serial roofline: every action of the plan
    # (first productions and recomputes) at max(FLOPs/TC peak, algorithmic
    # HBM bytes/HBM peak) — the time a speed-of-light kernel sequence needs
    step_roof = {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "tensor_bound_ms": 0.0, "hbm_bound_ms": 0.0,
                 "by_op": {}}
    for nid, lst in timing.items():
        if nid == "swap":
            for (ms, op, nb) in lst:
                swap_ms += ms
                swap_bytes += nb
                swap_n += 1
            continue
        node = rt.nodes[nid]
        for (ms, rec) in lst:
            t_tc = node.flops / (tc_peak * 1e9)
            t_mem = (node.hbm_bytes or 2 * node.nbytes) / (hbm_peak * 1e6)
            step_roof["ms"] += max(t_tc, t_mem)
            step_roof["flops"] += node.flops
            step_roof["bytes"] += node.hbm_bytes or 2 * node.nbytes
            step_roof["tensor_bound_ms" if t_tc >= t_mem else "hbm_bound_ms"] += max(t_tc, t_mem)
            bo = step_roof["by_op"].setdefault(node.op, [0.0, 0.0])
            bo[0] += ms
            bo[1] += max(t_tc, t_mem)
            all_ms += ms
            kinds[node.op] = kinds.get(node.op, 0.0) + ms
            if node.op == "conv":
                conv_ms += ms
                conv_flops += node.flops
                conv_n += 1
                conv_roof_ms += max(node.flops / (tc_peak * 1e9), node.hbm_bytes / (hbm_peak * 1e6))
            if rec:
                # recompute engine: each re-launch against its own roofline
                # (tensor-core FLOPs or HBM bytes, whichever bounds it)
                t_roof = max(node.flops / (tc_peak * 1e9), node.hbm_bytes / (hbm_peak * 1e6))
                rc["launches"] += 1
                rc["ms"] += ms
                bo = rc["by_op"].setdefault(node.op, [0, 0.0, 0.0])
                bo[0] += 1
                bo[1] += ms
                bo[2] += t_roof
                rc["roofline_ms"] += t_roof
                rc["flops"] += node.flops
                rc["bytes"] += node.hbm_bytes
    achieved = conv_flops / (conv_ms * 1e-3) / 1e12 if conv_ms else 0.0

    # ---- CPU baseline: the reference simulator planning this exact trace ----
    cpu = None
    if rank == 0:
        try:
            from oracle import ref as oref
            if oref.available():
                tj = trace.to_json()
                one = oref.time_run_ns(tj, rt.config, 5)
                iters = max(1, int(args.cpu_sample_s / max(one * 1e-9, 1e-6)))
                ns = oref.time_run_ns(tj, rt.config, iters)
                sim = oref.run(tj, rt.config)
                nproc, model = host_cpu()
                # the reference's answer for THIS run's trace (same costs,
                # budget, bandwidth): the step time its simulator predicts for
                # its plan, and what producing that plan costs on one core
                cpu = {"value": round(B / (sim["wall_time_us"] * 1e-6), 1), "unit": "images/s",
                       "cores": 1, "kind": "reference",
                       "sample": f"reference simulator on this run's {len(trace.nodes)}-node "
                                 f"ResNet-{args.depth} bs{B} trace: predicted step "
                                 f"{sim['wall_time_us']} us (simulated, not trained); "
                                 f"{iters} x run_iteration at {ns * 1e-3:.0f} us/plan on one "
                                 f"core of {nproc} ({model})",
                       "ms_per_plan": round(ns * 1e-6, 4),
                       "same_decisions": sim["decisions"] == [[n, int(a)] for n, a in prog.decisions]}
                try:  # the reference arm plans the committed fixture: same trace?
                    strip = lambda t: [{k: v for k, v in n.items() if k != "compute_cost_us"}
                                       for n in json.loads(t)["nodes"]]
                    fx = open(TRACE_FIXTURE).read()
                    cpu["fixture_same_structure"] = (strip(fx) == strip(tj) and
                                                     json.loads(fx)["schedule"] == json.loads(tj)["schedule"])
                except Exception:  # noqa: BLE001
                    pass
        except Exception as e:  # the baseline must never break the bench
            cpu = {"value": None, "unit": "images/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}
        ours_plan_ns = P.plan_time_ns(trace, rt.config, 200)

    # ---- max batch vs no-eviction in this GPU's HBM (planner-decided; the
    # ---- end-to-end verification is scripts/max_batch_verify.py) ----
    from paper_2203_15980_b200 import maxbatch as MB
    per_sample = {n.name: n.cost_us / B for n in rt.nodes}
    cap = free_hbm - 8 * 2**30  # persistent state + workspaces + slack
    bpus = int((rt.link_gbs or 50.0) * 1e3)
    mb_base = MB.search(args.depth, cap, per_sample, bpus, delta=False)
    mb_delta = {a: MB.search(args.depth, cap, per_sample, bpus, delta=True, anchors=a)
                for a in ("out+narrow", "out")}
    max_batch = {"no_eviction": mb_base.batch if mb_base else None,
                 "delta": {a: (f.batch if f else None) for a, f in mb_delta.items()},
                 "capacity_gb": round(cap / 1e9, 1)}
    best = max((f.batch for f in mb_delta.values() if f), default=None)
    if best and mb_base:
        max_batch["ratio"] = round(best / mb_base.batch, 3)
    # config 3: ResNet-101 (its extra layer3 blocks take layer3.1's per-sample costs)
    ps101 = MB.per_sample_costs(101, per_sample)
    b101 = MB.search(101, cap, ps101, bpus, delta=False)
    d101 = MB.search(101, cap, ps101, bpus, delta=True, anchors="out")
    max_batch["resnet101"] = {"no_eviction": b101.batch if b101 else None,
                              "delta": d101.batch if d101 else None,
                              "ratio": round(d101.batch / b101.batch, 3) if b101 and d101 else None}
    max_batch["note"] = ("planner-decided (arena + batch-proportional workspace <= capacity); "
                         "'verified': real training steps at those sizes in this run")

    bert = None
    if args.bert_batch > 0:
        bert = bert_section(args, world, rank, dp, barrier, max_over_ranks)

    # ---- config 3, verified: free this process's ResNet-50 bs256 state and
    # ---- train real steps at the planned max batches (DELTA and no eviction)
    budget_bytes, link_gbs = rt.config.budget, rt.link_gbs
    saved_graph = None
    if not args.no_verify_max_batch and world == 1 and best and mb_base:
        import gc
        a_best = max((a for a in mb_delta if mb_delta[a]), key=lambda a: mb_delta[a].batch)
        del rt
        gc.collect()
        torch.cuda.empty_cache()
        ver = {}
        for label, batch, anchors, delta in (("no_eviction", mb_base.batch, "out", False),
                                             ("delta", mb_delta[a_best].batch, a_best, True)):
            try:
                ver[label] = verify_batch(args.depth, batch, anchors, delta, per_sample, link_gbs,
                                          cap, MB)
            except Exception as e:  # noqa: BLE001 - reported, never fatal
                ver[label] = {"batch": batch, "error": str(e)[:200]}
            gc.collect()
            torch.cuda.empty_cache()
        max_batch["verified"] = ver
        ok = all("img_s" in v for v in ver.values())
        max_batch["verified_ratio"] = (round(ver["delta"]["batch"] / ver["no_eviction"]["batch"], 3)
                                       if ok else None)

    value = world * B / (delta_ms * 1e-3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(delta_ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (N(0,1) images 224x224x3 + uniform labels, random init)",
            "config": {"workload": f"ResNet-{args.depth} training step, batch {B}/GPU, "
                                   f"DELTA at {int(args.budget * 100)}% activation budget",
                       "global_batch": B * world, "image": 224, "budget_fraction": args.budget,
                       "budget_bytes": budget_bytes, "anchors": args.anchors,
                       "parallelism": f"dp{world}", "graph": graph_state,
                       "l2": "working set >> 126 MB L2 (no flush needed)"},
            "no_eviction": {"images_per_s": round(world * B / (base_ms * 1e-3), 1),
                            "ms_per_step": round(base_ms, 3),
                            "ratio": round(base_ms / delta_ms, 4),
                            "peak_act_gb": round(base_peak / 1e9, 3),
                            "arena_gb": round(base_arena / 1e9, 3)},
            "peak_act_gb": {"delta_report_peak": round(prog.plan_peak_bytes / 1e9, 3),
                            "delta_arena": round(prog.arena_bytes / 1e9, 3),
                            "no_eviction": round(base_peak / 1e9, 3),
                            "saving": round(1 - prog.arena_bytes / base_arena, 4)},
            "plan": {"counts": prog.plan_counts, "decisions": len(prog.decisions),
                     "host_slab_mb": round(prog.host_bytes / 2**20, 1),
                     "link_gbs": round(link_gbs, 2) if link_gbs else None,
                     "simulated_wall_us": prog.plan_wall_us,
                     "planner_ms": round(ours_plan_ns * 1e-6, 4)},
            "e2e": {"value": round(world * B / e2e_s, 1), "unit": "images/s",
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                    "loss_first_last": [round(losses[0], 4), round(losses[-1], 4)]},
            "roofline": {"kernel": "conv_fwd (tcgen05 implicit GEMM; forward + recompute)",
                         "bound": "tensor", "achieved": round(achieved, 1),
                         "peak": tc_peak, "unit": "TFLOP/s",
                         "frac": round(achieved / tc_peak, 4) if tc_peak else None,
                         "peak_kind": f"{peak_kind} burst bf16",
                         "traffic": conv_traffic.get("dram_bytes_per_launch"),
                         "traffic_note": conv_traffic.get("note"),
                         "launches_timed": conv_n,
                         "frac_of_roofline_time": round(conv_roof_ms / conv_ms, 4) if conv_ms else None,
                         "roofline_time_note": "sum over conv launches of max(FLOPs/TC peak, "
                                               "algorithmic bytes/HBM peak) / their device time "
                                               "(the 1x1 layer-1 convs are HBM-bound)",
                         "share_of_step": round(conv_ms / all_ms, 4) if all_ms else None,
                         "op_ms": {k: round(v, 3) for k, v in sorted(kinds.items(), key=lambda kv: -kv[1])}},
            "step_roofline": {"serial_roofline_ms": round(step_roof["ms"], 3),
                              "frac": round(step_roof["ms"] / delta_ms, 4),
                              "tflop": round(step_roof["flops"] / 1e12, 3),
                              "hbm_gb": round(step_roof["bytes"] / 1e9, 2),
                              "tensor_bound_ms": round(step_roof["tensor_bound_ms"], 3),
                              "hbm_bound_ms": round(step_roof["hbm_bound_ms"], 3),
                              "by_op_ms_vs_roofline": {k: [round(v[0], 3), round(v[1], 3)] for k, v in
                                                       sorted(step_roof["by_op"].items(),
                                                              key=lambda kv: kv[1][1] - kv[1][0])},
                              "note": "sum over every action of the DELTA step (incl. recomputes) "
                                      "of max(FLOPs/TC peak, algorithmic HBM bytes/HBM peak), "
                                      "vs the measured graph step (graph.py byte model)"},
            "recompute": {"launches": rc["launches"], "ms_per_step": round(rc["ms"], 3),
                          "share_of_step": round(rc["ms"] / all_ms, 4) if all_ms else None,
                          "roofline_ms": round(rc["roofline_ms"], 3),
                          "frac_of_roofline": round(rc["roofline_ms"] / rc["ms"], 4) if rc["ms"] else None,
                          "hbm_gb": round(rc["bytes"] / 1e9, 3),
                          "by_op": {k: {"n": v[0], "ms": round(v[1], 3),
                                        "frac_of_roofline": round(v[2] / v[1], 3) if v[1] else None}
                                    for k, v in rc["by_op"].items()},
                          "note": "eager step, CUDA events per recompute launch; roofline = "
                                  "max(FLOPs/TC peak, algorithmic bytes/HBM peak) per launch"},
            "swap": {"copies": swap_n, "bytes_per_step": swap_bytes,
                     "ms_per_step": round(swap_ms, 3),
                     "achieved_gbs": round(swap_bytes / (swap_ms * 1e6), 2) if swap_ms else None,
                     "link_probe_gbs": round(link_gbs, 2) if link_gbs else None,
                     "peak_gbs": PCIE5_X16_GBS,
                     "frac_of_link_peak": round(swap_bytes / (swap_ms * 1e6) / PCIE5_X16_GBS, 4)
                     if swap_ms else None,
                     "note": "copy-engine D2H/H2D on their own streams (events on those streams); "
                             "peak = PCIe Gen5 x16 nominal per direction"},
            "max_batch": max_batch,
            "cpu_baseline": cpu,
            "gpu_launches": launches * args.steps,
            "clocks": clk,
            "parity": parity,
            "bert": bert,
        }
        detail = line
        # the full record goes to a side file; the printed line keeps the
        # headline keys short enough to survive a log tail
        dpath = args.detail or os.path.join(
            HERE, "gpurun_out" if os.path.isdir(os.path.join(HERE, "gpurun_out")) else "",
            "bench_detail.json")
        try:
            with open(dpath, "w") as f:
                json.dump(detail, f, indent=1)
        except OSError:
            dpath = None
        rf = detail["roofline"]
        mb = detail["max_batch"]
        line = {k: detail[k] for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                                        "ms_per_step", "higher_is_better", "scaling",
                                        "vs_baseline", "dtype", "data")}
        line.update({
            "config": {k: detail["config"][k] for k in ("workload", "global_batch", "budget_bytes",
                                                          "parallelism", "graph", "l2")},
            "parity": parity,
            "no_eviction_ratio": detail["no_eviction"]["ratio"],
            "no_eviction_images_per_s": detail["no_eviction"]["images_per_s"],
            "peak_act_gb": detail["peak_act_gb"]["delta_arena"],
            "peak_act_gb_no_eviction": detail["peak_act_gb"]["no_eviction"],
            "max_batch_ratio": mb.get("ratio"),
            "max_batch": {"no_eviction": mb["no_eviction"], "delta": max(
                (v for v in mb["delta"].values() if v), default=None),
                "resnet101_ratio": mb["resnet101"]["ratio"],
                "kind": "trained" if mb.get("verified_ratio") else "planner-decided",
                "verified_ratio": mb.get("verified_ratio")},
            "plan": detail["plan"]["counts"],
            "e2e": {k: detail["e2e"][k] for k in ("value", "unit", "h2d_bytes_per_step",
                                                   "d2h_bytes_per_step")},
            "roofline": {k: rf[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
            "roofline_kernel": "conv_fwd tcgen05 (fwd+recompute)",
            "step_roofline_frac": detail["step_roofline"]["frac"],
            "recompute_roofline_frac": detail["recompute"]["frac_of_roofline"],
            "swap_gbs": detail["swap"]["achieved_gbs"],
            "cpu_baseline": ({k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
                             if cpu else None),
            "gpu_launches": detail["gpu_launches"],
            "clocks": clk,
            "bert": ({k: bert[k] for k in ("seq_per_s", "tokens_per_s", "ms_per_step",
                                            "no_eviction_ratio", "peak_act_gb",
                                            "peak_act_gb_no_eviction", "parity", "model_tflops")}
                     | {"e2e_seq_per_s": bert["e2e"]["seq_per_s"],
                        "workload": f"BERT-large seq 512 bs{args.bert_batch}/GPU, "
                                    f"{int(args.bert_budget * 100)}% budget (config 5)"}
                     if bert else None),
            "detail": os.path.relpath(dpath, HERE) if dpath else None,
        })
        print(json.dumps(line), flush=True)
    if dp is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
