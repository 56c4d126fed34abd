"""Stress run behind DESIGN.md §12: fresh contexts in a warm process, the multislice call on device and pinned
outputs, every slice against warm single calls (usage: flake_hunt.py [reps])."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_13431_b200 as K
from paper_2302_13431_b200 import phantom
case = phantom.generate("C3", slices=14, full_dims=(64, 64), channels=8)
spec = case.spec
cfg = K.PipelineConfig(kernel=spec.kernel, tau=spec.tau, nullspace_threshold=spec.nullspace_threshold,
                       power_iters=spec.power_iters, grid=K.GRID_REDUCED, grid_pad=spec.grid_dims[0] - spec.calib[0])
s, q, full = case.calib.shape[0], spec.channels, spec.full_dims
# warm the process with other work (module loading, other kernels)
c2 = phantom.generate("C1")
ctxw = K.Context(0)
for _ in range(2):
    K.estimate_maps(K.Calib(c2.calib[0], c2.center_offset), c2.spec.full_dims,
                    K.PipelineConfig(kernel=c2.spec.kernel, tau=c2.spec.tau, power_iters=c2.spec.power_iters,
                                     grid=K.GRID_REDUCED, grid_pad=c2.spec.grid_dims[0] - c2.spec.calib[0]), ctxw,
                    want_spectrum=False)
ctxr = K.Context(0)
ref = [K.estimate_maps(K.Calib(case.calib[i], case.center_offset), full, cfg, ctxr, want_spectrum=False) for i in range(s)]
refm = np.stack([r.maps for r in ref]); refl = np.stack([r.lambda_min_map for r in ref])
cal = torch.from_numpy(case.calib).cuda()
bad = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    ctx = K.Context(0)
    for kind in ("dev", "pin", "pin2"):
        if kind == "dev":
            bufs = [torch.empty((s, q) + full, dtype=torch.complex64, device="cuda"),
                    torch.empty((s,) + full, dtype=torch.float32, device="cuda"),
                    torch.empty((s,) + full, dtype=torch.uint8, device="cuda")]
        else:
            bufs = [torch.full((s, q) + full, 3 + 3j, dtype=torch.complex64).pin_memory(),
                    torch.full((s,) + full, -1.0, dtype=torch.float32).pin_memory(),
                    torch.full((s,) + full, 7, dtype=torch.uint8).pin_memory()]
        torch.cuda.synchronize()
        pv = K.api.estimate_maps_batched_device(ctx, cal.data_ptr(), s, spec.calib, case.center_offset, q, full, cfg,
                                                bufs[0].data_ptr(), bufs[1].data_ptr(), bufs[2].data_ptr())
        m = bufs[0].cpu().numpy(); l = bufs[1].cpu().numpy()
        for i in range(s):
            d = np.linalg.norm(m[i] - refm[i]) / np.linalg.norm(refm[i])
            if d > 1e-5:
                bad += 1
                dm = np.abs(m[i] - refm[i]).max(0)
                rows = np.where(dm.max(1) > 1e-4)[0]
                print(f"rep {rep} {kind} slice {i}: maps rel {d:.3e} rank {int(pv[i].nullspace_rank)} ref {ref[i].nullspace_rank} "
                      f"its {int(pv[i].subspace_iterations)} b {int(pv[i].subspace_block)} lam diff {np.abs(l[i]-refl[i]).max():.3e} "
                      f"rows affected {len(rows)} [{rows.min() if len(rows) else -1}..{rows.max() if len(rows) else -1}]", flush=True)
    ctx.close()
print("bad slices:", bad)
