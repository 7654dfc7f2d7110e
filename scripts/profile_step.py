"""One eager DELTA training step of ResNet-50 bs256 @50% between
cudaProfilerStart/Stop, for `ncu --profile-from-start off`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200.runtime import DeltaRuntime  # noqa: E402

B = int(os.environ.get("PB", "256"))
rt = DeltaRuntime(50, B, seed=0)
rt.plan(0.5)
for _ in range(2):
    rt.step_device()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
rt.step_device()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled one step", rt.program.plan_counts)
