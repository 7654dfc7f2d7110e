"""Trace capture from a PyTorch training step (§8 f1, paper_2203_15980_b200/
capture.py): the captured trace is a valid deltasim Trace, it has the DELTA
structure (uncomputable batch, forward activations read by backward ops), and
on it our planner's decisions and timeline equal the reference simulator's."""
import hashlib

import pytest
import torch
import torch.nn as nn
import torch.nn.functional as F

from paper_2203_15980_b200 import capture as CAP
from paper_2203_15980_b200 import planner as P


def _model():
    torch.manual_seed(0)
    return nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.BatchNorm2d(16), nn.ReLU(),
                         nn.Conv2d(16, 32, 3, padding=1, stride=2), nn.BatchNorm2d(32), nn.ReLU(),
                         nn.Conv2d(32, 32, 3, padding=1), nn.BatchNorm2d(32), nn.ReLU(),
                         nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(32, 10))


@pytest.fixture(scope="module")
def captured():
    x = torch.randn(8, 3, 32, 32)
    y = torch.randint(0, 10, (8,))
    return CAP.capture_trace(_model(), (x, y), lambda out, x, y: F.cross_entropy(out, y),
                             name="cnn", timing=True)


def test_captured_trace_is_valid(captured):
    t, nodes = captured
    assert t.validate()[0] == 0
    # round trip through the reference's JSON schema (parse_trace)
    t2 = P.Trace.from_json(t.to_json())
    assert len(t2.nodes) == len(t.nodes) and len(t2.schedule) == len(t.schedule)


def test_captured_trace_structure(captured):
    t, nodes = captured
    assert t.nodes[0].uncomputable and t.nodes[0].evict_pinned      # the batch
    assert t.nodes[1].uncomputable                                   # the labels
    assert t.nodes[0].output_bytes == 8 * 3 * 32 * 32 * 4
    fwd = [e.node for e in t.schedule if e.phase == P.Phase.Forward]
    bwd = [e.node for e in t.schedule if e.phase == P.Phase.Backward]
    assert len(fwd) >= 12 and len(bwd) >= 10
    names = {n.id: n.name for n in t.nodes}
    assert sum("convolution." in names[i] for i in fwd) == 3
    assert sum("convolution_backward" in names[i] for i in bwd) >= 2
    # backward ops read saved forward activations (ReLU masks, BN inputs)
    fset = set(fwd)
    relu_bwd = [n for n in t.nodes if "threshold_backward" in n.name]
    assert relu_bwd and all(any(p in fset for p in n.parents) for n in relu_bwd)
    assert all(n.compute_cost_us >= 1 for n in t.nodes)


@pytest.mark.parametrize("frac", [0.7, 0.85, 1.0])
@pytest.mark.parametrize("mode", [P.PolicyMode.Delta, P.PolicyMode.RecomputeOnly])
def test_plan_on_captured_trace_matches_reference(captured, frac, mode):
    oracle_ref = pytest.importorskip("oracle.ref")
    if not oracle_ref.available():
        pytest.skip("oracle/_ref not built")
    t, _ = captured
    base = P.run_unconstrained_baseline(t, P.EngineConfig())
    cfg = P.EngineConfig(budget=int(base.peak_bytes * frac), policy_mode=mode)
    mine = P.run_iteration(t, cfg)
    ref = oracle_ref.run(t.to_json(), cfg)
    assert ref["decisions"] == [[n, int(a)] for n, a in mine.decisions]
    assert ref["chrome"] == mine.chrome_trace()
    assert ref["peak_bytes"] == mine.peak_bytes
