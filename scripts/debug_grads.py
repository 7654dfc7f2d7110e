import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn.functional as F
from paper_2203_15980_b200.runtime import DeltaRuntime
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from test_runtime_gpu import make_batch
torch.backends.cudnn.deterministic = True
rt = DeltaRuntime(50, 16, seed=0, lr=0.0)
rt.plan(None)
x, y = make_batch(0)
names = ["fc.bwd", "layer4.2.bn3.bwd", "layer4.2.conv3.bwd", "layer4.2.conv2.bwd", "layer4.2.conv1.bwd", "layer4.1.bn3.bwd",
         "layer4.2.conv2", "layer4.2.bn2_relu", "layer4.2.conv3", "layer4.2.out", "avgpool"]
ids = {rt.g.node(n).id: n for n in names}
probe = {i: None for i in ids}
rt.x_dev.copy_(x); rt.y_dev.copy_(y)
with torch.cuda.stream(rt.stream):
    rt.run_program(probe=probe)
torch.cuda.synchronize()
print("loss", rt.loss.item())
# reference with retained intermediates
pr = rt.params
params = {k: v.detach().clone().requires_grad_(True) for k, v in pr.views.items()}
acts = {}
def keep(name, t):
    t.retain_grad(); acts[name] = t; return t
h = x.float().cuda().permute(0, 3, 1, 2)
def conv(name, t):
    cs = rt.g.convs[name]; return F.conv2d(t, params["conv:" + name].permute(0, 3, 1, 2), stride=cs.stride, padding=cs.pad)
def bn(name, t):
    return F.batch_norm(t, None, None, params["bn_g:" + name], params["bn_b:" + name], training=True, eps=1e-5)
h = F.relu(bn("bn1", conv("conv1", h))); h = F.max_pool2d(h, 3, 2, 1)
for li, nb in enumerate([3, 4, 6, 3]):
    for b in range(nb):
        pre = f"layer{li+1}.{b}"
        c1 = keep(pre+".conv1", conv(pre + ".conv1", h))
        o = F.relu(bn(pre + ".bn1", c1))
        c2 = keep(pre+".conv2", conv(pre + ".conv2", o))
        o = keep(pre+".bn2_relu", F.relu(bn(pre + ".bn2", c2)))
        c3 = keep(pre+".conv3", conv(pre + ".conv3", o))
        o = bn(pre + ".bn3", c3)
        sc = bn(pre + ".downsample.1", conv(pre + ".downsample.0", h)) if b == 0 else h
        h = keep(pre+".out", F.relu(o + sc))
pooled = keep("avgpool", h.mean((2, 3)))
logits = pooled @ params["fc_w"].t() + params["fc_b"]
loss = F.cross_entropy(logits, y.cuda()); loss.backward()
print("ref loss", loss.item())
def cos(a, b):
    a = a.flatten().float(); b = b.flatten().float()
    return F.cosine_similarity(a, b, dim=0).item(), (a.norm()/b.norm()).item()
def nhwc(t): return t.permute(0, 2, 3, 1) if t.dim() == 4 else t
pairs = [("fc.bwd", acts["avgpool"].grad), ("layer4.2.bn3.bwd", nhwc(acts["layer4.2.conv3"].grad)),
         ("layer4.2.conv3.bwd", nhwc(acts["layer4.2.conv2"].grad)), ("layer4.2.conv2.bwd", nhwc(acts["layer4.2.conv1"].grad)),
         ("layer4.2.conv1.bwd", nhwc(acts["layer4.1.out"].grad)),
         ("layer4.2.conv2", nhwc(acts["layer4.2.conv2"])), ("layer4.2.bn2_relu", nhwc(acts["layer4.2.bn2_relu"])),
         ("layer4.2.conv3", nhwc(acts["layer4.2.conv3"])), ("layer4.2.out", nhwc(acts["layer4.2.out"])), ("avgpool", acts["avgpool"])]
for n, ref in pairs:
    print(n, cos(probe[rt.g.node(n).id], ref))
for name in ["conv:layer4.2.conv3", "conv:layer4.2.conv2", "conv:layer4.2.conv1", "bn_g:layer4.2.bn3", "bn_b:layer4.2.bn3", "bn_g:layer4.2.bn2"]:
    print(name, cos(pr.gviews[name], params[name].grad))
