import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn.functional as F
from paper_2203_15980_b200.runtime import DeltaRuntime
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from test_runtime_gpu import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rt = DeltaRuntime(50, B, seed=0, lr=0.0)
rt.plan(None)
x, y = make_batch(0, B)
probe = {n.id: None for n in rt.nodes if n.phase == "F"}
rt.x_dev.copy_(x); rt.y_dev.copy_(y)
with torch.cuda.stream(rt.stream):
    rt.run_program(probe=probe)
torch.cuda.synchronize()
pr = rt.params
P = {k: v.detach().float() for k, v in pr.views.items()}
ref = {}
def conv(name, t):
    cs = rt.g.convs[name]; return F.conv2d(t, P["conv:" + name].permute(0, 3, 1, 2), stride=cs.stride, padding=cs.pad)
def bn(name, t):
    return F.batch_norm(t, None, None, P["bn_g:" + name], P["bn_b:" + name], training=True, eps=1e-5)
def ours(name):  # NHWC bf16 -> NCHW fp32
    t = probe[rt.g.node(name).id].float()
    return t.permute(0, 3, 1, 2) if t.dim() == 4 else t
def cmp(name, r):
    o = ours(name)
    c = F.cosine_similarity(o.flatten(), r.flatten(), dim=0).item()
    print(f"{name:28s} cos={c:.6f} maxerr={(o - r).abs().max().item():.4g} refmax={r.abs().max().item():.4g}", flush=True)
# reference evaluated op by op FROM OUR OWN INPUTS (isolates each kernel)
xin = ours("input")
cmp("conv1", conv("conv1", xin[:, :3] if False else xin))
cmp("bn1_relu", F.relu(bn("bn1", ours("conv1"))))
cmp("maxpool", F.max_pool2d(ours("bn1_relu"), 3, 2, 1))
h = "maxpool"
for li, nb in enumerate([3, 4, 6, 3]):
    for b in range(nb):
        pre = f"layer{li+1}.{b}"
        cmp(pre + ".conv1", conv(pre + ".conv1", ours(h)))
        cmp(pre + ".bn1_relu", F.relu(bn(pre + ".bn1", ours(pre + ".conv1"))))
        cmp(pre + ".conv2", conv(pre + ".conv2", ours(pre + ".bn1_relu")))
        cmp(pre + ".bn2_relu", F.relu(bn(pre + ".bn2", ours(pre + ".conv2"))))
        cmp(pre + ".conv3", conv(pre + ".conv3", ours(pre + ".bn2_relu")))
        if b == 0:
            cmp(pre + ".downsample.0", conv(pre + ".downsample.0", ours(h)))
            sc = bn(pre + ".downsample.1", ours(pre + ".downsample.0"))
        else:
            sc = ours(h)
        cmp(pre + ".out", F.relu(bn(pre + ".bn3", ours(pre + ".conv3")) + sc))
        h = pre + ".out"
cmp("avgpool", ours(h).mean((2, 3)))
