"""Multi-process host logic of the slice sharding (C3), on CPU with gloo.

Two ranks each generate only their block of slices, run the per-slice
estimator (the FP64 oracle here: no GPU in the CPU suite), and all-gather the
outputs; the reassembled result must equal the single-process run bit for bit.
"""
import os
import socket

import numpy as np
import pytest

from paper_2302_13431_b200 import shard


def test_partition_covers_disjoint_balanced():
    for n in (0, 1, 5, 128, 129):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard.partition(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.partition(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASE = dict(name="C3", slices=5, full_dims=(32, 32), channels=4)


def _estimate(calib, center_offset, spec):
    from oracle import oracle as O
    cfg = O.PipelineConfig.pisco()
    cfg.tau, cfg.power_iters, cfg.grid = 2, 8, O.GRID_FULL
    r = O.estimate_maps(O.Calib(calib.astype(np.complex128), center_offset), spec.full_dims, cfg)
    return {"maps": r.maps.astype(np.complex64), "lambda": r.lambda_min_map.astype(np.float32),
            "mask": r.support_mask}


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from paper_2302_13431_b200 import phantom
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = CASE["slices"]
    a, b = shard.partition(n, world, rank)
    case = phantom.generate(CASE["name"], slices=n, full_dims=CASE["full_dims"], channels=CASE["channels"],
                            slice_range=(a, b))
    local = shard.run_local(lambda c: _estimate(c, case.center_offset, case.spec), list(case.calib))
    for key in ("maps", "lambda", "mask"):
        arr = local.get(key)
        if arr is None:  # a rank with no slices still participates in the gather
            ref = _estimate(case.calib[0] if len(case.calib) else np.zeros(
                (CASE["channels"],) + case.spec.calib, np.complex64), case.center_offset, case.spec)[key]
            arr = np.zeros((0,) + ref.shape, ref.dtype)
        full = shard.gather_slices(arr, n)
        if rank == 0:
            np.save(os.path.join(out_dir, f"{key}.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_gather_equals_single_process(tmp_path):
    import torch.multiprocessing as mp
    from paper_2302_13431_b200 import phantom
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    n = CASE["slices"]
    case = phantom.generate(CASE["name"], slices=n, full_dims=CASE["full_dims"], channels=CASE["channels"])
    ref = shard.run_local(lambda c: _estimate(c, case.center_offset, case.spec), list(case.calib))
    for key in ("maps", "lambda", "mask"):
        got = np.load(tmp_path / f"{key}.npy")
        assert got.shape == ref[key].shape
        assert np.array_equal(got, ref[key]), key


def test_slice_data_independent_of_partition():
    from paper_2302_13431_b200 import phantom
    full = phantom.generate("C3", slices=6, full_dims=(32, 32), channels=4)
    part = phantom.generate("C3", slices=6, full_dims=(32, 32), channels=4, slice_range=(3, 6))
    assert np.array_equal(full.calib[3:], part.calib)


# --------------------------------------------------------------- C4: z-slabs
ZS = dict(full=(12, 10, 10), grid=(8, 8, 6), calib=(6, 6, 6), q=3)


class _OracleOps:
    """The z-slab driver's operations on the FP64 oracle (CPU tensors)."""

    def __init__(self, calib, cfg_o):
        from oracle import oracle as O
        self.O = O
        res = O.estimate_maps(O.Calib(calib.data.astype(np.complex128), calib.center_offset), ZS["full"], cfg_o,
                              grid_dims=ZS["grid"], want_raw=True)
        self.norm = O.normalize_maps(res.raw_maps, O.Calib(calib.data.astype(np.complex128),
                                                           calib.center_offset))[0].astype(np.complex64)
        self.lam = res.raw_lambda.astype(np.float32)
        self.final = res

    def raw_slab(self, calib, full_dims, cfg, slab):
        import torch
        a, b = slab
        return torch.from_numpy(self.norm[:, a:b].copy()), torch.from_numpy(self.lam[a:b].copy())

    # the broadcast path: root computes the signal basis, every rank expands it
    allow_basis = True
    basis_seen = None

    def signal_basis(self, calib, cfg):
        import torch
        assert self.allow_basis, "only the root computes the nullspace"
        O = self.O
        cal = O.Calib(calib.data.astype(np.complex128), calib.center_offset)
        g = O.gram_fft(cal, cfg.kernel, cfg.tau)
        w, v = np.linalg.eigh(g)  # nullspace.cpp:13-33 in complement form
        sig = np.sqrt(np.maximum(w, 0.0))
        keep = sig >= cfg.nullspace_threshold * sig[-1]
        u = v[:, keep]
        return {"u": torch.from_numpy(u.copy()), "n": g.shape[0], "k": int(keep.sum()), "sigma1": float(sig[-1]),
                "rank": int(g.shape[0] - keep.sum())}

    def raw_slab_basis(self, calib, full_dims, cfg, slab, basis):
        import torch
        O = self.O
        self.basis_seen = basis
        u = basis["u"].numpy()
        q = calib.channels
        W = np.eye(u.shape[0]) - u @ u.conj().T  # aggregate_w of the complement basis
        field = O.gram_field_fast(W, q, cfg.kernel, cfg.tau, ZS["grid"])
        lam = O.make_support(cfg.kernel, cfg.tau, 3).shape[0]
        vec, val = O.eig_power_field(O.espirit(field, lam), cfg.power_iters)
        raw = vec.reshape((q,) + ZS["grid"])
        norm = O.normalize_maps(raw, O.Calib(calib.data.astype(np.complex128), calib.center_offset))[0]
        a, b = slab
        lamr = (1.0 - val).reshape(ZS["grid"])
        return (torch.from_numpy(norm[:, a:b].astype(np.complex64).copy()),
                torch.from_numpy(lamr[a:b].astype(np.float32).copy()))

    def interpolate_maps(self, low, full_dims):
        import torch
        return torch.from_numpy(self.O.interpolate_maps(low.numpy(), full_dims).astype(np.complex64))

    def interpolate_real(self, low, full_dims):
        import torch
        return torch.from_numpy(self.O.interpolate_real(low.numpy(), full_dims).astype(np.float32))

    def sos_accumulate(self, maps, sos):
        sos += (maps.real ** 2 + maps.imag ** 2).sum(0)
        return sos

    def renormalize(self, maps, sos):
        import torch
        pos = sos > 0
        maps[:, pos] = maps[:, pos] / torch.sqrt(sos[pos])
        return maps

    def support_mask(self, lam, thr):
        return (lam < thr).to(dtype=__import__("torch").uint8)


def _zs_case():
    from oracle import oracle as O
    from paper_2302_13431_b200 import api as A
    sc = O.simulate(ZS["q"], ZS["full"], 1, 5, noise_sigma=0.01, noise_seed=3)
    cal = O.extract_calibration(sc["kspace"], ZS["calib"])
    calib = A.Calib(cal.data.astype(np.complex64), tuple(cal.center_offset))
    ck = A.PipelineConfig(kernel=A.ELLIPSOID, tau=1, power_iters=12, grid_dims=ZS["grid"])
    co = O.PipelineConfig.pisco()
    co.tau, co.power_iters = 1, 12
    return calib, ck, co


def _zs_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calib, ck, co = _zs_case()
    ops = _OracleOps(calib, co)
    ops.allow_basis = rank == 0  # the other ranks must receive the filters by broadcast
    maps, lam, mask, info = shard.estimate_maps_zslab(calib, ZS["full"], ck, ops)
    np.save(os.path.join(out_dir, f"basis{rank}.npy"), ops.basis_seen["u"].numpy())
    if rank == 0:
        np.save(os.path.join(out_dir, "maps.npy"), maps.numpy())
        np.save(os.path.join(out_dir, "lam.npy"), lam.numpy())
        np.save(os.path.join(out_dir, "mask.npy"), mask.numpy())
    np.save(os.path.join(out_dir, f"slab{rank}.npy"), np.array(info["slab"]))
    dist.barrier()
    dist.destroy_process_group()


def test_zslab_two_rank_gloo_equals_single_process(tmp_path):
    """SURVEY §8e for C4: z-slab G(x)/power iteration per rank, all-gather of the
    low-resolution maps, channel-split interpolation with an all-reduced SoS.
    Two gloo ranks must reproduce the single-process composition and the
    oracle's own finalize (maps.cpp:236-258)."""
    import torch.multiprocessing as mp
    mp.spawn(_zs_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    calib, ck, co = _zs_case()
    ops = _OracleOps(calib, co)
    maps1, lam1, mask1, _ = shard.estimate_maps_zslab(calib, ZS["full"], ck, ops)
    maps2 = np.load(tmp_path / "maps.npy")
    assert [tuple(np.load(tmp_path / f"slab{r}.npy")) for r in range(2)] == [(0, 4), (4, 8)]
    u0, u1 = np.load(tmp_path / "basis0.npy"), np.load(tmp_path / "basis1.npy")
    assert np.array_equal(u0, u1)  # rank 1 expanded exactly the root's broadcast filters
    assert maps2.shape == maps1.shape == (ZS["q"],) + ZS["full"]
    assert np.allclose(maps2, maps1.numpy(), rtol=1e-5, atol=1e-6)
    assert np.array_equal(np.load(tmp_path / "lam.npy"), lam1.numpy())
    assert np.array_equal(np.load(tmp_path / "mask.npy"), mask1.numpy())
    ref = ops.final  # the oracle's own interpolate + renormalise + mask
    num = np.linalg.norm(maps2 - ref.maps)
    assert num / np.linalg.norm(ref.maps) < 1e-5
    assert np.allclose(np.load(tmp_path / "lam.npy"), ref.lambda_min_map, rtol=1e-5, atol=1e-7)
