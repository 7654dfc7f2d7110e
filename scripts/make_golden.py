"""Regenerate tests/golden/ from the UNMODIFIED reference (oracle/_ref, built by
`make -C oracle` from /root/reference/proj/src).  Run in the build container:

    python scripts/make_golden.py

Outputs (all produced by the reference binary, none hand-written):
  resnet16.json / linear8.json            gen_resnet_like(16,1<<20,0) / gen_linear_chain(8,100,5,0)
  resnet16_delta50_report.json            report_to_json(summarize(run @ peak/2, baseline))
  linear8_baseline_timeline.json          chrome trace of linear8, Baseline, budget 800
  ref_vectors.json                        reference run_iteration outputs (decisions, counts,
                                          peak, wall, stall, sha256 of the chrome trace) for
                                          fuzzed DAG traces x configs, the bundled fixtures
                                          and the ResNet-50 bs256 trace at 40/50/60 %
"""
import hashlib
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2203_15980_b200 import planner as P  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")


def fuzz_trace(rng: random.Random, max_nodes: int, max_bytes=1000, max_cost=50) -> str:
    """Random DAG, node 0 an uncomputable input, <= 3 parents, forward produce
    then reverse backward use (the reference's fuzz shape, tests/helpers.hpp:46-79),
    plus optional pins and backward produce nodes to reach the other paths."""
    n = rng.randint(2, max_nodes)
    nodes = []
    for i in range(n):
        parents = []
        if i > 0:
            for _ in range(rng.randint(1, min(i, 3))):
                p = rng.randrange(i)
                if p not in parents:
                    parents.append(p)
        unc = i == 0
        ep = unc or rng.random() < 0.08
        op = (not unc) and rng.random() < 0.08
        nodes.append(dict(id=i, name=f"n{i}", compute_cost_us=rng.randint(1, max_cost),
                          output_bytes=rng.randint(1, max_bytes), parents=parents,
                          uncomputable=unc, evict_pinned=ep, offload_pinned=op))
    sched = [dict(node=i, phase="F", kind="P") for i in range(n)]
    back = []
    nb = rng.randint(0, 3)
    for j in range(nb):  # backward-produced gradient nodes
        nid = n + j
        ps = sorted(set(rng.randrange(n) for _ in range(rng.randint(1, 3))))
        nodes.append(dict(id=nid, name=f"g{j}", compute_cost_us=rng.randint(1, max_cost),
                          output_bytes=rng.randint(1, max_bytes), parents=ps,
                          uncomputable=False, evict_pinned=False, offload_pinned=False))
    for i in range(n - 1, -1, -1):
        back.append(dict(node=i, phase="B", kind="U"))
    for j in range(nb):
        back.insert(rng.randrange(len(back) + 1), dict(node=n + j, phase="B", kind="P"))
    return json.dumps(dict(name="fuzz", nodes=nodes, schedule=sched + back),
                      separators=(",", ":"))


def cfg_variants(rng: random.Random, peak: int):
    for _ in range(4):
        c = P.EngineConfig(budget=max(1, int(peak * rng.choice([0.35, 0.5, 0.6, 0.75, 1.0]))))
        c.policy_mode = P.PolicyMode(rng.choice([0, 0, 0, 1, 2]))
        c.heuristic = P.Heuristic(rng.randrange(3))
        c.cost_model = P.CostModel(bandwidth_bytes_per_us=rng.choice([(64000, 1), (50, 1), (3, 2)]),
                                   effective_fraction=rng.choice([(7, 20), (1, 1), (1, 3)]),
                                   swap_cost_mode=P.SwapCostMode(rng.randrange(2)))
        c.watermark_fraction = rng.choice([(3, 4), (1, 1), (1, 2), (2, 3)])
        c.prefetch_limit = rng.choice([0, 1, 2, 3])
        c.prefetch_enabled = rng.random() < 0.8
        c.overlap_enabled = rng.random() < 0.8
        c.prefetch_guard = P.PrefetchGuard(rng.randrange(2))
        yield c


def cfg_dict(c):
    return dict(budget=c.budget, heuristic=int(c.heuristic), policy=int(c.policy_mode),
                bw=list(c.cost_model.bandwidth_bytes_per_us), eff=list(c.cost_model.effective_fraction),
                swap_mode=int(c.cost_model.swap_cost_mode), wm=list(c.watermark_fraction),
                prefetch_limit=c.prefetch_limit, prefetch_enabled=c.prefetch_enabled,
                overlap_enabled=c.overlap_enabled, guard=int(c.prefetch_guard))


def summary(out: dict) -> dict:
    if not out.get("ok"):
        return dict(error=out.get("what", "")[:80])
    return dict(decisions=out["decisions"], counts=out["counts"], peak=out["peak_bytes"],
                wall=out["wall_time_us"], stall=out["total_stall_us"],
                infeasible=out["infeasible"], n_events=len(out["events"]),
                chrome_sha256=hashlib.sha256(out["chrome"].encode()).hexdigest())


def main():
    assert ref.available(), "build oracle/_ref first: make -C oracle"
    os.makedirs(G, exist_ok=True)
    r16 = ref.generate("resnet", 16, 0)
    l8 = ref.generate("linear", 8, 0)
    open(os.path.join(G, "resnet16.json"), "w").write(r16)
    open(os.path.join(G, "linear8.json"), "w").write(l8)
    base = ref.run(r16, P.EngineConfig(), baseline=True)
    open(os.path.join(G, "resnet16_delta50_report.json"), "w").write(
        ref.report(r16, P.EngineConfig(budget=base["peak_bytes"] // 2)))
    lin = ref.run(l8, P.EngineConfig(budget=800, policy_mode=P.PolicyMode.Baseline))
    open(os.path.join(G, "linear8_baseline_timeline.json"), "w").write(lin["chrome"])

    vectors = []
    rng = random.Random(20261017)
    for t in range(160):
        tj = fuzz_trace(rng, rng.choice([6, 12, 30, 60]))
        peak = ref.run(tj, P.EngineConfig(), baseline=True)
        if not peak.get("ok"):
            continue
        for c in cfg_variants(rng, peak["peak_bytes"]):
            vectors.append(dict(trace=tj, cfg=cfg_dict(c), ref=summary(ref.run(tj, c))))
    for name, tj in [("resnet16", r16), ("linear8", l8)]:
        pk = ref.run(tj, P.EngineConfig(), baseline=True)["peak_bytes"]
        for frac in (0.4, 0.5, 0.6):
            for h in range(3):
                c = P.EngineConfig(budget=int(pk * frac), heuristic=P.Heuristic(h))
                vectors.append(dict(trace=name, cfg=cfg_dict(c), ref=summary(ref.run(tj, c))))
    r50 = open(os.path.join(G, "resnet50_bs256_trace.json")).read()
    meta = json.load(open(os.path.join(G, "resnet50_bs256_trace.meta.json")))
    pk = ref.run(r50, P.EngineConfig(), baseline=True)["peak_bytes"]
    for frac in (0.4, 0.5, 0.6):
        c = P.EngineConfig(budget=int(pk * frac), cost_model=P.CostModel(
            bandwidth_bytes_per_us=tuple(meta["bandwidth_bytes_per_us"]), effective_fraction=(1, 1)))
        vectors.append(dict(trace="resnet50_bs256_trace", cfg=cfg_dict(c), ref=summary(ref.run(r50, c))))
    with open(os.path.join(G, "ref_vectors.json"), "w") as f:
        json.dump(vectors, f, separators=(",", ":"))
    print(f"wrote {len(vectors)} reference vectors")


if __name__ == "__main__":
    main()
