"""Multi-process sharding with the REAL GPU ops, two ranks on one GPU.

The box has one GPU, so both ranks hold their own sk_ctx on cuda:0 and talk
over gloo (host collectives; no kernel of one rank waits on the other).  The
data path is the one bench.py drives on N GPUs:

* C3-style slice sharding: each rank runs the batched multislice call on its
  block of slices, one all-gather reassembles them; the result must equal the
  single-process batched run and match the FP64 oracle.
* C4-style z-slabs: rank 0 runs K1 + K2 and broadcasts U_sig (the nullspace
  filters in complement form), each rank expands G(x) and iterates only its
  slab, all-gather of the low-resolution maps, channel-split interpolation with
  an all-reduced SoS; compared with the unsharded GPU pipeline and the oracle.
"""
import os
import socket

import numpy as np
import pytest

from tests import parity as PM

pytestmark = pytest.mark.gpu

MS = dict(slices=5, full=(64, 64), channels=8, tau=3, grid=(48, 48), iters=20)
ZS = dict(full=(24, 24, 16), grid=(16, 16, 12), calib=(10, 10, 10), q=4, tau=1, iters=12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ms_case():
    from paper_2302_13431_b200 import phantom
    return phantom.generate("C3", slices=MS["slices"], full_dims=MS["full"], channels=MS["channels"])


def _ms_cfg(K):
    return K.PipelineConfig(kernel=K.ELLIPSOID, tau=MS["tau"], power_iters=MS["iters"], grid=K.GRID_REDUCED,
                            grid_pad=MS["grid"][0] - 24)


def _zs_case():
    from oracle import oracle as O
    import paper_2302_13431_b200 as K
    sc = O.simulate(ZS["q"], ZS["full"], 1, 7, noise_sigma=0.01, noise_seed=5)
    cal = O.extract_calibration(sc["kspace"], ZS["calib"])
    calib = K.Calib(cal.data.astype(np.complex64), tuple(cal.center_offset))
    ck = K.PipelineConfig(kernel=K.ELLIPSOID, tau=ZS["tau"], power_iters=ZS["iters"], grid_dims=ZS["grid"])
    return calib, ck


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    import paper_2302_13431_b200 as K
    from paper_2302_13431_b200 import phantom, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = K.Context(0)
    # --- slice sharding
    a, b = shard.partition(MS["slices"], world, rank)
    case = phantom.generate("C3", slices=MS["slices"], full_dims=MS["full"], channels=MS["channels"],
                            slice_range=(a, b))
    maps, lam, mask, provs = K.api.estimate_maps_batched(case.calib, case.center_offset, MS["full"], _ms_cfg(K), ctx)
    full_maps = shard.gather_slices(maps, MS["slices"])
    full_lam = shard.gather_slices(lam, MS["slices"])
    ranks = shard.gather_slices(np.array([p["rank"] for p in provs], dtype=np.int64), MS["slices"])
    # --- z-slabs with the broadcast basis, device tensors
    calib, ck = _zs_case()
    ops = shard.DeviceOps(ctx, torch.device("cuda", 0))
    zm, zl, zk, info = shard.estimate_maps_zslab(calib, ZS["full"], ck, ops)
    if rank == 0:
        np.save(os.path.join(out_dir, "ms_maps.npy"), full_maps)
        np.save(os.path.join(out_dir, "ms_lam.npy"), full_lam)
        np.save(os.path.join(out_dir, "ms_rank.npy"), ranks)
        np.save(os.path.join(out_dir, "zs_maps.npy"), zm.cpu().numpy())
        np.save(os.path.join(out_dir, "zs_lam.npy"), zl.cpu().numpy())
        np.save(os.path.join(out_dir, "zs_info.npy"), np.array([info["k"], info["rank"]]))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_two_rank_sharding_on_gpu_ops(tmp_path):
    import torch.multiprocessing as mp
    import paper_2302_13431_b200 as K
    from oracle import oracle as O
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)

    # slice sharding == single-process batched run == oracle
    case = _ms_case()
    ctx = K.Context(0)
    maps1, lam1, mask1, provs1 = K.api.estimate_maps_batched(case.calib, case.center_offset, MS["full"], _ms_cfg(K),
                                                             ctx)
    got = np.load(tmp_path / "ms_maps.npy")
    assert np.array_equal(np.load(tmp_path / "ms_rank.npy"), [p["rank"] for p in provs1])
    for s in range(MS["slices"]):
        assert PM.maps_nrmse(got[s], maps1[s], mask1[s]) < 1e-6
    co = O.PipelineConfig.pisco()
    co.tau, co.power_iters, co.grid_pad = MS["tau"], MS["iters"], MS["grid"][0] - 24
    for s in (0, MS["slices"] - 1):
        ref = O.estimate_maps(O.Calib(case.calib[s].astype(np.complex128), case.center_offset), MS["full"], co)
        assert PM.maps_nrmse(got[s], ref.maps, ref.support_mask) < PM.TOL_MAPS
        assert PM.lambda_errors(np.load(tmp_path / "ms_lam.npy")[s], ref.lambda_min_map)["normwise"] < PM.TOL_LAMBDA

    # z-slabs with the broadcast basis == unsharded GPU pipeline == oracle
    calib, ck = _zs_case()
    res = K.estimate_maps(calib, ZS["full"], ck, ctx, want_spectrum=False)
    zm = np.load(tmp_path / "zs_maps.npy")
    k, r = np.load(tmp_path / "zs_info.npy")
    assert r == res.nullspace_rank
    assert PM.maps_nrmse(zm, res.maps, res.support_mask) < 1e-5
    assert PM.lambda_errors(np.load(tmp_path / "zs_lam.npy"), res.lambda_min_map)["normwise"] < 1e-5
    co = O.PipelineConfig.pisco()
    co.tau, co.power_iters = ZS["tau"], ZS["iters"]
    ref = O.estimate_maps(O.Calib(calib.data.astype(np.complex128), calib.center_offset), ZS["full"], co,
                          grid_dims=ZS["grid"])
    assert r == ref.nullspace_rank
    assert PM.maps_nrmse(zm, ref.maps, ref.support_mask) < PM.TOL_MAPS
    ctx.close()
