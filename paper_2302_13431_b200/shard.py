"""Multi-GPU plumbing for the sharded configurations.

Multislice 2-D (C3) is a set of independent estimate_maps problems, one per
slice: slices are split into contiguous blocks across ranks (one process per
GPU) and every rank runs the whole pipeline (its own Gram, eigensolve, G(x),
power iteration) on its block.  There is no data-path collective; the only
communication is an optional gather of the per-slice outputs to rank 0
(NCCL over NVLink on the box, gloo in the CPU tests).  Single-slice configs
(C1, C2, C5) do not shard: ranks run independent replicas.
"""
from __future__ import annotations

import numpy as np


def partition(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of `n_items` for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def counts(n_items: int, world: int) -> list[int]:
    return [b - a for a, b in (partition(n_items, world, r) for r in range(world))]


def run_local(estimate_one, calibs_local):
    """Apply `estimate_one(calib) -> dict of arrays` to each local slice; stack per key."""
    outs = [estimate_one(c) for c in calibs_local]
    if not outs:
        return {}
    return {k: np.stack([o[k] for o in outs]) for k in outs[0]}


def gather_slices(local: np.ndarray, n_items: int, group=None, device=None):
    """Gather per-rank slice blocks (leading axis = slices) to every rank, in slice order.

    Uses all_gather over equal-size padded blocks (the block sizes differ by at
    most one); returns the concatenated (n_items, ...) array on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = counts(n_items, world)
    pad = max(cnt)
    shape = local.shape[1:]
    buf = np.zeros((pad,) + shape, dtype=local.dtype)
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf.view(np.uint8).reshape(pad, -1).copy())
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    rows = []
    for r, p in enumerate(parts):
        arr = p.cpu().numpy().reshape((pad,) + (-1,)).view(local.dtype).reshape((pad,) + shape)
        rows.append(arr[: cnt[r]])
    return np.concatenate(rows, axis=0)


# --------------------------------------------------------------- C4: z-slabs
# A 3-D volume shards by z-slab (axis 0 of the map grid).  The root rank runs
# the Gram and the nullspace once and BROADCASTS the nullspace filters in
# their complement form U_sig (n x k; W = I - U_sig U_sig^H, C4: 3936 x 37
# complex128 = 2.3 MB) together with k and sigma_1 (north_star);
# every rank expands G(x) from that same basis and runs the power iteration +
# normalisation only on its rows of the map grid (sk_estimate_raw_slab_basis);
# one all-gather assembles the low-resolution maps and eigenvalues; the
# interpolation is split by channel, its sum-of-squares renormalisation by an
# all-reduce of the per-voxel SoS (maps.cpp:236-258).  Tensors stay where the
# ops put them (HBM with NCCL on the box, host memory with gloo in the CPU
# tests; a gloo group with CUDA tensors stages them through the host).

def _is_gloo(group=None):
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _staged(t, group=None):
    """Tensor to hand to a collective: host copy for gloo + CUDA tensors."""
    return t.cpu() if (t.is_cuda and _is_gloo(group)) else t


def broadcast_basis(basis, root: int = 0, group=None, device=None):
    """Broadcast the root's signal basis {"u": (n, k) complex128, "k", "sigma1",
    "rank", "n"} to every rank (two collectives: the sizes, then U_sig)."""
    import torch
    import torch.distributed as dist
    me = dist.get_rank(group)
    meta = torch.zeros(4, dtype=torch.float64, device=device)
    if me == root:
        meta = torch.tensor([basis["n"], basis["k"], basis["sigma1"], basis["rank"]], dtype=torch.float64,
                            device=device)
    m = _staged(meta, group)
    dist.broadcast(m, root, group=group)
    n, k, sigma1, rank = int(m[0]), int(m[1]), float(m[2]), int(m[3])
    if me == root:
        u = torch.view_as_real(basis["u"].contiguous()).contiguous()
    else:
        u = torch.empty((n, k, 2), dtype=torch.float64, device=device)
    us = _staged(u, group)
    dist.broadcast(us, root, group=group)
    if us is not u:
        u.copy_(us)
    return {"u": torch.view_as_complex(u), "n": n, "k": k, "sigma1": sigma1, "rank": rank}

def _gather_rows(t, n_total: int, group=None):
    """all_gather of per-rank row blocks (dim 0, sizes from partition) -> (n_total, ...) on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = counts(n_total, world)
    pad = max(cnt)
    real = torch.view_as_real(t) if t.is_complex() else t
    buf = _staged(real.new_zeros((pad,) + tuple(real.shape[1:])), group)
    buf[: real.shape[0]] = real.to(buf.device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat([p[:c] for p, c in zip(parts, cnt)], 0).to(real.device)
    return torch.view_as_complex(out.contiguous()) if t.is_complex() else out


class DeviceOps:
    """The z-slab driver's operations on the C-ABI with device tensors."""

    def __init__(self, ctx, device):
        self.ctx, self.device = ctx, device

    def _ready(self):
        """The library runs on the context's own non-blocking stream: tensors
        that torch kernels just produced (transposes, fills, slices made
        contiguous) must be complete before a C-ABI call reads them."""
        import torch
        torch.cuda.current_stream(self.device).synchronize()

    def _cal(self, calib):
        import torch
        cal = calib.data if isinstance(calib.data, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(calib.data, dtype=np.complex64))
        return cal.to(self.device).contiguous()

    def raw_slab(self, calib, full_dims, cfg, slab):
        """K1 + K2 + the slab's K3/K4/normalisation on this rank (no broadcast)."""
        import torch
        from . import api
        grid = api._grid_for(calib.dims, full_dims, cfg)
        q = calib.channels
        shape = (slab[1] - slab[0],) + tuple(grid[1:])
        cal = self._cal(calib)
        maps = torch.empty((q,) + shape, dtype=torch.complex64, device=self.device)
        lam = torch.empty(shape, dtype=torch.float32, device=self.device)
        self._ready()
        api.estimate_raw_slab_device(self.ctx, cal.data_ptr(), calib.dims, calib.center_offset, q, full_dims, cfg,
                                     slab, maps.data_ptr(), lam.data_ptr())
        return maps, lam

    def signal_basis(self, calib, cfg):
        """compute_gram + extract_nullspace on this rank -> the signal basis dict."""
        import torch
        from . import api
        cal = self._cal(calib)
        q = calib.channels
        n = q * api.make_support(cfg.kernel, cfg.tau, len(calib.dims)).shape[0]
        kmax = min(n, 256)
        while True:
            u = torch.empty((kmax, n), dtype=torch.complex128, device=self.device)  # column-major n x kmax
            self._ready()
            try:
                info = api.signal_basis_device(self.ctx, cal.data_ptr(), calib.dims, calib.center_offset, q, cfg,
                                               u.data_ptr(), kmax)
                break
            except api.DimError:
                if kmax >= n:
                    raise
                kmax = n
        k = info["k"]
        return {"u": u[:k].transpose(0, 1), "n": n, "k": k, "sigma1": info["sigma1"], "rank": info["rank"]}

    def raw_slab_basis(self, calib, full_dims, cfg, slab, basis):
        """The slab's K3/K4/normalisation from a (broadcast) signal basis."""
        import torch
        from . import api
        grid = api._grid_for(calib.dims, full_dims, cfg)
        q = calib.channels
        shape = (slab[1] - slab[0],) + tuple(grid[1:])
        cal = self._cal(calib)
        u = basis["u"].transpose(0, 1).contiguous().to(self.device)  # (k, n) row-major = n x k column-major
        maps = torch.empty((q,) + shape, dtype=torch.complex64, device=self.device)
        lam = torch.empty(shape, dtype=torch.float32, device=self.device)
        self._ready()
        api.estimate_raw_slab_basis_device(self.ctx, cal.data_ptr(), calib.dims, calib.center_offset, q, full_dims,
                                           cfg, u.data_ptr(), basis["k"], basis["sigma1"], slab, maps.data_ptr(),
                                           lam.data_ptr())
        return maps, lam

    def interpolate_maps(self, low, full_dims):
        import ctypes as C
        import torch
        from . import api
        low = low.contiguous()
        out = torch.empty((low.shape[0],) + tuple(full_dims), dtype=torch.complex64, device=low.device)
        self._ready()
        api._check(api.lib().sk_interpolate_maps(self.ctx.handle, low.dim() - 1, api._p(api._i64(low.shape[1:])),
                                                 low.shape[0], C.c_void_p(low.data_ptr()),
                                                 api._p(api._i64(full_dims)), C.c_void_p(out.data_ptr())))
        return out

    def interpolate_real(self, low, full_dims):
        import ctypes as C
        import torch
        from . import api
        low = low.contiguous()
        out = torch.empty(tuple(full_dims), dtype=torch.float32, device=low.device)
        self._ready()
        api._check(api.lib().sk_interpolate_real(self.ctx.handle, low.dim(), api._p(api._i64(low.shape)),
                                                 C.c_void_p(low.data_ptr()), api._p(api._i64(full_dims)),
                                                 C.c_void_p(out.data_ptr())))
        return out

    def sos_accumulate(self, maps, sos):
        from . import api
        self._ready()
        return api.sos_accumulate(maps, sos, self.ctx)

    def renormalize(self, maps, sos):
        from . import api
        self._ready()
        return api.renormalize_sos(maps, sos, self.ctx)

    def support_mask(self, lam, thr):
        import ctypes as C
        import torch
        from . import api
        out = torch.empty(lam.shape, dtype=torch.uint8, device=lam.device)
        self._ready()
        api._check(api.lib().sk_support_mask(self.ctx.handle, lam.numel(), C.c_void_p(lam.data_ptr()), float(thr),
                                             C.c_void_p(out.data_ptr())))
        return out


def estimate_maps_zslab(calib, full_dims, cfg, ops, group=None, gather_maps=True):
    """estimate_maps (maps.cpp:265-330) sharded by z-slab across the ranks of `group`.

    Returns (maps, lambda, mask, info): maps (Q, *full) when gather_maps else
    this rank's channel block (info["channels"]); lambda and mask on every rank.
    """
    import torch
    import torch.distributed as dist
    from . import api

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    grid = api._grid_for(calib.dims, full_dims, cfg)
    q = calib.channels
    slab = partition(grid[0], world, rank)
    if world > 1:
        # the exchange step: root's K1 + K2 once, its filters broadcast to every rank
        basis = ops.signal_basis(calib, cfg) if rank == 0 else None
        basis = broadcast_basis(basis, 0, group, device=getattr(ops, "device", None))
        maps_s, lam_s = ops.raw_slab_basis(calib, full_dims, cfg, slab, basis)  # (Q, nz, ...), (nz, ...)
    else:
        maps_s, lam_s = ops.raw_slab(calib, full_dims, cfg, slab)
    if world > 1:
        maps_low = _gather_rows(maps_s.transpose(0, 1).contiguous(), grid[0], group).transpose(0, 1).contiguous()
        lam_low = _gather_rows(lam_s, grid[0], group)
    else:
        maps_low, lam_low = maps_s, lam_s
    ch = partition(q, world, rank)
    if tuple(grid) == tuple(full_dims):  # no interpolation, no renormalisation (maps.cpp:236-237)
        mine = maps_low[ch[0]:ch[1]].contiguous()
        lam = lam_low
    else:
        mine = ops.interpolate_maps(maps_low[ch[0]:ch[1]].contiguous(), full_dims)
        sos = torch.zeros(tuple(full_dims), dtype=torch.float32, device=mine.device)
        ops.sos_accumulate(mine, sos)
        if world > 1:
            ss = _staged(sos, group)
            dist.all_reduce(ss, group=group)
            if ss is not sos:
                sos.copy_(ss)
        ops.renormalize(mine, sos)
        lam = ops.interpolate_real(lam_low, full_dims)
    mask = ops.support_mask(lam, cfg.mask_threshold)
    maps = _gather_rows(mine, q, group) if (gather_maps and world > 1) else mine
    info = {"slab": slab, "channels": ch, "grid": grid}
    if world > 1:
        info.update(k=basis["k"], rank=basis["rank"], sigma1=basis["sigma1"])
    return maps, lam, mask, info
