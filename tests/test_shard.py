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
