"""One warm C2 estimate_maps for profiling (device buffers)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_13431_b200 as K
from paper_2302_13431_b200 import phantom
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
case = phantom.generate(name)
spec = case.spec
cfg = K.PipelineConfig(kernel=spec.kernel, tau=spec.tau, power_iters=spec.power_iters,
                       grid=K.GRID_FULL if spec.full_grid else K.GRID_REDUCED,
                       grid_pad=spec.grid_dims[0] - spec.calib[0], grid_dims=spec.grid_dims if spec.ndim == 3 else None)
ctx = K.Context(0)
cal = torch.from_numpy(case.calib[0]).cuda()
q = spec.channels
maps = torch.empty((q,) + spec.full_dims, dtype=torch.complex64, device="cuda")
lam = torch.empty(spec.full_dims, dtype=torch.float32, device="cuda")
mask = torch.empty(spec.full_dims, dtype=torch.uint8, device="cuda")
for i in range(steps):
    p = K.api.estimate_maps_device(ctx, cal.data_ptr(), spec.calib, case.center_offset, q, spec.full_dims, cfg,
                                   maps.data_ptr(), lam.data_ptr(), mask.data_ptr())
    print(i, [round(x, 3) for x in p.stage_ms], round(p.total_ms, 3), "iters", p.subspace_iterations, "b", p.subspace_block, flush=True)
