"""§8 f1/f3/f4 on a B200: capture DELTA traces of PyTorch training steps (ATen
level, device-timed costs) and plan them with libdelta over a budget x policy
grid (the paper's Fig. 8 analogue; acceptance C8).  Config 5: BERT-large
(24 layers, hidden 1024, 16 heads, FFN 4096) at seq 512, bf16, 40 % budget.
Plans are checked against the reference simulator on the same trace.
Writes gpurun_out/capture_models.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import capture as CAP  # noqa: E402
from paper_2203_15980_b200 import kernels as K  # noqa: E402
from paper_2203_15980_b200 import planner as P  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dev = torch.device("cuda")
link = min(K.probe_link()[:2])
cm = P.CostModel((int(link * 1e3), 1), (1, 1))
try:
    from oracle import ref as oref
    have_ref = oref.available()
except Exception:  # noqa: BLE001
    have_ref = False


def grid(t, name):
    base = P.run_unconstrained_baseline(t, P.EngineConfig(cost_model=cm))
    rows = []
    for frac in (0.3, 0.4, 0.5, 0.7):
        for mode in (P.PolicyMode.Delta, P.PolicyMode.RecomputeOnly, P.PolicyMode.OffloadOnly):
            cfg = P.EngineConfig(budget=int(base.peak_bytes * frac), policy_mode=mode, cost_model=cm)
            r = P.run_iteration(t, cfg)
            row = dict(budget_frac=frac, policy=mode.name, feasible=r.completed(),
                       counts=r.counts, peak_gb=round(r.peak_bytes / 1e9, 3),
                       sim_wall_ms=round(r.wall_time_us / 1e3, 3),
                       slowdown=round(r.wall_time_us / base.wall_time_us, 4),
                       stall_ms=round(r.total_stall_us / 1e3, 3))
            if have_ref:
                ref = oref.run(t.to_json(), cfg)
                row["reference_identical"] = (ref["decisions"] == [[n, int(a)] for n, a in r.decisions]
                                              and ref["chrome"] == r.chrome_trace())
            rows.append(row)
    return dict(model=name, nodes=len(t.nodes), events=len(t.schedule),
                baseline_peak_gb=round(base.peak_bytes / 1e9, 3),
                baseline_wall_ms=round(base.wall_time_us / 1e3, 3), grid=rows)


out = {"link_gbs": round(link, 2), "models": []}

# ---- BERT-large, seq 512 (config 5 shape), synthetic tokens, MLM-style loss ----
from transformers import BertConfig, BertModel  # noqa: E402
cfg = BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                 intermediate_size=4096, max_position_embeddings=512, vocab_size=30522)
torch.manual_seed(0)
bert = BertModel(cfg).to(dev, torch.bfloat16).train()
B, S = 8, 512
ids = torch.randint(0, cfg.vocab_size, (B, S), device=dev)
t, _ = CAP.capture_trace(bert, (ids,), lambda out, ids: out.last_hidden_state.float().pow(2).mean(),
                         name="bert_large_s512_b8")
res = grid(t, f"BERT-large seq{S} bs{B} bf16")
out["models"].append(res)
print(json.dumps({k: v for k, v in res.items() if k != "grid"}), flush=True)
for row in res["grid"]:
    print(json.dumps(row), flush=True)
del bert
torch.cuda.empty_cache()

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "capture_models.json"), "w"), indent=1)
