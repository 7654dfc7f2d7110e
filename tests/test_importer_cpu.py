"""PyTorch CNN -> DELTA graph the runtime executes (SURVEY 8(f) f1,
paper_2203_15980_b200/importer.py): the graph is a valid trace whose plans
match the reference simulator's, every node has a kernel recipe type, and
what the kernels cannot run is refused (no fallback)."""
import pytest
import torch.nn as nn

from paper_2203_15980_b200 import graph as G
from paper_2203_15980_b200 import importer as IM
from paper_2203_15980_b200 import planner as P

RECIPE_OPS = {"input", "conv", "bn_relu", "maxpool", "avgpool", "fc", "fc_bwd", "bn_add_relu_bwd",
              "conv_bn_relu_bwd", "conv_bwd", "maxpool_bwd", "bn_relu_bwd", "conv_wgrad"}


def small_cnn(num_classes=10):
    """stem + maxpool, 4 x 3x3/64, a stride-2 3x3, 3 x 3x3/128, a 1x1 to 256, head"""
    layers = [nn.Conv2d(3, 64, 7, 2, 3, bias=False), nn.BatchNorm2d(64), nn.ReLU(),
              nn.MaxPool2d(3, 2, 1)]
    for _ in range(4):
        layers += [nn.Conv2d(64, 64, 3, 1, 1, bias=False), nn.BatchNorm2d(64), nn.ReLU()]
    layers += [nn.Conv2d(64, 128, 3, 2, 1, bias=False), nn.BatchNorm2d(128), nn.ReLU()]
    for _ in range(3):
        layers += [nn.Conv2d(128, 128, 3, 1, 1, bias=False), nn.BatchNorm2d(128), nn.ReLU()]
    layers += [nn.Conv2d(128, 256, 1, bias=False), nn.BatchNorm2d(256), nn.ReLU(),
               nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(256, num_classes)]
    return nn.Sequential(*layers)


def test_imported_graph_is_a_valid_trace_with_recipes():
    model = small_cnn()
    g, names = IM.graph_from_module(model, batch=32, image=224)
    assert {n.op for n in g.nodes} <= RECIPE_OPS
    assert {"conv_bwd", "maxpool_bwd", "bn_relu_bwd", "conv_bn_relu_bwd", "conv_wgrad"} <= \
        {n.op for n in g.nodes}
    n_conv = sum(isinstance(m, nn.Conv2d) for m in model)
    assert len(names["conv"]) == n_conv == len(names["bn"]) and names["fc"] == str(len(model) - 1)
    t = G.to_trace(g)
    assert t.validate()[0] == 0
    assert g.convs["c5"].stride == 2 and g.fc == (256, 10) and g.fc_pad == 64
    # every backward node reads only earlier nodes
    for n in g.nodes:
        assert all(p < n.id for p in n.parents)


@pytest.mark.parametrize("frac", [0.5, 0.7, 0.85])
def test_imported_graph_plans_match_reference(frac):
    ref = pytest.importorskip("oracle.ref")
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    g, _ = IM.graph_from_module(small_cnn(), batch=32, image=224)
    t = G.to_trace(g)
    base = P.run_unconstrained_baseline(t, P.EngineConfig())
    cfg = P.EngineConfig(budget=int(base.peak_bytes * frac))
    mine = P.run_iteration(t, cfg)
    out = ref.run(t.to_json(), cfg)
    assert out["decisions"] == [[n, int(a)] for n, a in mine.decisions]
    assert out["chrome"] == mine.chrome_trace()


@pytest.mark.parametrize("bad,msg", [
    (lambda: nn.Sequential(nn.Conv2d(3, 16, 3, padding=1, bias=False), nn.BatchNorm2d(16), nn.ReLU(),
                           nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(16, 10)), "stem"),
    (lambda: nn.Sequential(nn.Conv2d(3, 64, 7, 2, 3), nn.BatchNorm2d(64), nn.ReLU(),
                           nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(64, 10)), "bias-free"),
    (lambda: nn.Sequential(nn.Conv2d(3, 64, 7, 2, 3, bias=False), nn.BatchNorm2d(64),
                           nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(64, 10)), "BatchNorm2d and ReLU"),
    (lambda: nn.Sequential(nn.Conv2d(3, 64, 7, 2, 3, bias=False), nn.BatchNorm2d(64), nn.ReLU(),
                           nn.Conv2d(64, 96, 3, 1, 1, bias=False), nn.BatchNorm2d(96), nn.ReLU(),
                           nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(96, 10)), "power of two"),
    (lambda: nn.Sequential(nn.Conv2d(3, 64, 7, 2, 3, bias=False), nn.BatchNorm2d(64), nn.ReLU(),
                           nn.Dropout(), nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(64, 10)),
     "unsupported module"),
])
def test_unsupported_models_are_refused(bad, msg):
    with pytest.raises(IM.UnsupportedModel, match=msg):
        IM.graph_from_module(bad(), batch=8, image=64)


def test_residual_model_refused():
    class Res(nn.Module):
        def __init__(self):
            super().__init__()
            self.c = nn.Conv2d(64, 64, 3, 1, 1, bias=False)

        def forward(self, x):
            return x + self.c(x)
    with pytest.raises(IM.UnsupportedModel):
        IM.graph_from_module(Res(), batch=8, image=32, in_channels=64)
