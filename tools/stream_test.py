import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2302_13431_b200 as K
from paper_2302_13431_b200 import phantom
case = phantom.generate("C2"); spec = case.spec
cfg = K.PipelineConfig(kernel=spec.kernel, tau=spec.tau, nullspace_threshold=spec.nullspace_threshold, power_iters=spec.power_iters,
                       grid=K.GRID_FULL if spec.full_grid else K.GRID_REDUCED, grid_pad=spec.grid_dims[0] - spec.calib[0])
for mode in sys.argv[1:]:
    ctx = K.Context(0)
    if mode == "torch":
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    elif mode == "side":
        s = torch.cuda.Stream(); ctx.set_stream(s.cuda_stream)
    cal = torch.from_numpy(case.calib[0]).cuda()
    q = spec.channels
    maps = torch.empty((q,) + spec.full_dims, dtype=torch.complex64, device="cuda")
    lam = torch.empty(spec.full_dims, dtype=torch.float32, device="cuda")
    mask = torch.empty(spec.full_dims, dtype=torch.uint8, device="cuda")
    for i in range(6):
        p = K.api.estimate_maps_device(ctx, cal.data_ptr(), spec.calib, case.center_offset, q, spec.full_dims, cfg,
                                       maps.data_ptr(), lam.data_ptr(), mask.data_ptr())
    print(mode, [round(x, 3) for x in p.stage_ms], round(p.total_ms, 3), "stream", torch.cuda.current_stream().cuda_stream, flush=True)
