#!/bin/bash
# One ncu --set full capture of the whole-plane DMMA 2D DST (N = 31, 32 MB stack):
# tensor-pipe (DMMA) utilisation for the profiles (run on the GPU box).
cd "$(dirname "$0")/.."
ncu --set full --clock-control none -k regex:dmma_dst2d -c 1 -o gpurun_out/dmma_full \
  python -c "
import sys, torch
sys.path.insert(0, '.')
from paper_1912_03565_b200 import _native
lib = _native.load_library(); lib.hfb_set_tuning(18, 32)
n = 31; nz = (32 << 20) // (n * n)
plan = _native.get_plan(n, n, nz, torch.device('cuda', 0))
x = torch.randn((nz, n, n), dtype=torch.float64, device='cuda'); w = plan.workspace(1)
_native.check(lib.hfb_transform_stack(plan.handle, _native.ptr(x), 0, nz, _native.ptr(w), plan.stream()), 't')
torch.cuda.synchronize()
"
