#!/bin/bash
# ncu evidence for the DMMA / FFT crossover (run on the GPU box):
#   launch lists of the 2D transform of a 32 MB stack at N = 31 and 63, FFT engine
#   (tuning key 18 = 0) against the whole-plane DMMA kernel (key 18 = 64), and one
#   --set full capture of the DMMA kernel at N = 31.
set -e
cd "$(dirname "$0")/.."
for n in 31 63; do
  for k in 0 64; do
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed_op_dmma.sum \
        --clock-control none --csv --log-file gpurun_out/dmma_n${n}_k${k}.csv \
        python -c "
import sys, torch
sys.path.insert(0, '.')
from paper_1912_03565_b200 import _native
lib = _native.load_library(); lib.hfb_set_tuning(18, $k)
n = $n; nz = (32 << 20) // (n * n)
plan = _native.get_plan(n, n, nz, torch.device('cuda', 0))
x = torch.randn((nz, n, n), dtype=torch.float64, device='cuda'); w = plan.workspace(1)
_native.check(lib.hfb_transform_stack(plan.handle, _native.ptr(x), 0, nz, _native.ptr(w), plan.stream()), 't')
torch.cuda.synchronize()
" > /dev/null 2>&1
  done
done
