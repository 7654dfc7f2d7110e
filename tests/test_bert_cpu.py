"""The BERT-large DELTA graph (ref src/trace.cpp:422-466 op
set) on the CPU: it is a valid deltasim trace with the reference
transformer's per-layer structure, our planner's decisions / timeline on it
equal the reference simulator's at the config-5 budget (40 %) and around
it, and the host-built token CSR of the word-embedding gradient is right."""
import numpy as np
import pytest

from paper_2203_15980_b200 import bert as B
from paper_2203_15980_b200 import graph as G
from paper_2203_15980_b200 import planner as P


@pytest.fixture(scope="module")
def large():
    g = B.build_bert(B.BertConfig(batch=8))
    G.estimate_costs(g)
    return g, G.to_trace(g)


def test_bert_trace_structure(large):
    g, t = large
    assert t.validate()[0] == 0
    fwd = [n for n in g.nodes if n.phase == "F"]
    # embedding + 10 per layer + final LN + head
    assert len(fwd) == 1 + 24 * 10 + 2
    per_layer = [n.op for n in fwd[1:11]]
    # ref gen_transformer_like: LN1, QKV, Attention, OutProj, AddResid1, LN2, MlpUp, MlpDown,
    # AddResid2 (+ the GELU node between MlpUp and MlpDown)
    assert per_layer == ["layernorm", "linear", "attention", "linear", "add_dropout", "layernorm",
                         "linear", "gelu", "linear", "add_dropout"]
    T, H = 8 * 512, 1024
    assert fwd[3].nbytes == T * H * 2 and fwd[2].nbytes == 3 * T * H * 2
    assert fwd[7].nbytes == 4 * T * H * 2 and fwd[8].nbytes == 4 * T * H * 2
    # every backward node reads at least one saved activation or gradient
    assert all(n.parents for n in g.nodes if n.phase == "B")
    P.Trace.from_json(t.to_json())


@pytest.mark.parametrize("frac", [0.3, 0.4, 0.5])
@pytest.mark.parametrize("mode", [P.PolicyMode.Delta, P.PolicyMode.RecomputeOnly,
                                  P.PolicyMode.OffloadOnly])
def test_bert_plan_matches_reference(large, frac, mode):
    oracle_ref = pytest.importorskip("oracle.ref")
    if not oracle_ref.available():
        pytest.skip("oracle/_ref not built")
    _, t = large
    cm = P.CostModel(bandwidth_bytes_per_us=(55000, 1), effective_fraction=(1, 1))
    base = P.run_unconstrained_baseline(t, P.EngineConfig(cost_model=cm))
    cfg = P.EngineConfig(budget=int(base.peak_bytes * frac), policy_mode=mode, cost_model=cm)
    mine = P.run_iteration(t, cfg)
    ref = oracle_ref.run(t.to_json(), cfg)
    assert ref["decisions"] == [[n, int(a)] for n, a in mine.decisions]
    assert ref["chrome"] == mine.chrome_trace()
    assert ref["peak_bytes"] == mine.peak_bytes
    if mode == P.PolicyMode.Delta and frac == 0.4:
        assert not mine.infeasible and mine.counts["recompute"] > 0


def test_token_csr():
    ids = np.array([5, 3, 5, 9, 3, 5, 0])
    csr = B.token_csr(ids)
    T = ids.size
    U = csr[0]
    uniq, seg, perm = csr[1:1 + U], csr[1 + T:2 + T + U], csr[2 + 2 * T:]
    assert list(uniq) == [0, 3, 5, 9]
    for u, v in enumerate(uniq):
        idx = perm[seg[u]:seg[u + 1]]
        assert list(idx) == sorted(idx) and all(ids[idx] == v)
    assert sorted(perm) == list(range(T))
