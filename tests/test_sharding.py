"""Multi-rank logic on CPU: gloo, world size 2.

The GPU kernels are not run here; the tests pin what crosses the
interconnect: the packed-key MIN all-reduce of obstacle shards must pick the
same (d, link, voxel) as one rank seeing every voxel (lowest rank, then lowest
link on ties; -1/-1 at the clamp), and waypoint shards gather back in order.
"""

import os
import socket

import numpy as np
import pytest

from paper_2309_12543_b200 import sharding as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _reference_min(vals, clamp):
    """vals: (C, V, L) candidate values; first-min over (voxel, link) with the clamp rule."""
    C, V, L = vals.shape
    d = np.full(C, np.float32(clamp), np.float32)
    link = np.full(C, -1, np.int32)
    voxel = np.full(C, -1, np.int32)
    for c in range(C):
        best = None
        for v in range(V):
            for l in range(L):
                x = vals[c, v, l]
                if best is None or x < best[0]:
                    best = (x, v, l)
        if best[0] < np.float32(clamp):
            d[c], voxel[c], link[c] = best
    return d, link, voxel


def _shard_result(vals, lo, hi, clamp):
    d, link, voxel = _reference_min(vals[:, lo:hi], clamp)
    return d, link, voxel


def _worker(rank, world, port, vals, clamp, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    C, V, L = vals.shape
    lo, hi = S.shard_range(V, rank, world)
    d, link, voxel = _shard_result(vals, lo, hi, clamp)
    keys = S.pack_keys(d, link, voxel, L, voxel_offset=lo)
    red = S.unpack_keys(S.allreduce_min_keys(keys), L, clamp)
    # the tensor form the NCCL path runs on the device (here: gloo on host tensors)
    import torch

    kt = S.pack_keys_tensor(torch.from_numpy(d), torch.from_numpy(link), torch.from_numpy(voxel), L, voxel_offset=lo)
    dist.all_reduce(kt, op=dist.ReduceOp.MIN)
    red_t = tuple(x.numpy() for x in S.unpack_keys_tensor(kt, L, clamp))
    assert all(np.array_equal(a, b) for a, b in zip(red, red_t))
    wl, wh = S.shard_range(C, rank, world)
    gd, gl, gv = S.gather_waypoint_results(red[0][wl:wh], red[1][wl:wh], red[2][wl:wh])
    if rank == 0:
        out.put((red, (gd, gl, gv)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [0, 1])
def test_obstacle_shards_min_allreduce_gloo(seed):
    import multiprocessing as mp

    rng = np.random.default_rng(seed)
    C, V, L = 37, 23, 5
    vals = np.round(rng.normal(0.1, 0.1, size=(C, V, L)) * 64).astype(np.float32) / 64  # many exact ties
    vals[3] = 0.5                                   # everything above the clamp
    vals[4] = np.float32(0.3)                       # exactly the clamp -> -1/-1
    vals[5, :, :] = 0.25
    vals[5, 17, 2] = 0.0
    vals[5, 9, 4] = -0.0                            # -0.0 ties +0.0: rank 9 wins
    clamp = 0.3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, vals, clamp, q)) for r in range(2)]
    for p in procs:
        p.start()
    (d, link, voxel), (gd, gl, gv) = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rd, rl, rv = _reference_min(vals, clamp)
    assert np.array_equal(d, rd) and np.array_equal(link, rl) and np.array_equal(voxel, rv)
    assert link[3] == -1 and link[4] == -1 and voxel[5] == 9 and link[5] == 4
    assert np.array_equal(gd, rd) and np.array_equal(gl, rl) and np.array_equal(gv, rv)


def test_key_round_trip_and_order():
    d = np.float32([0.1, -0.2, 0.0, -0.0, 0.3, 1e-30])
    link = np.int32([1, 0, 2, 3, -1, 0])
    voxel = np.int32([5, 7, 1, 1, -1, 0])
    k = S.pack_keys(d, link, voxel, 4, voxel_offset=10)
    d2, l2, v2 = S.unpack_keys(k, 4, 0.3)
    assert np.array_equal(l2, link) and np.array_equal(v2[link >= 0], voxel[link >= 0] + 10)
    assert np.all(d2[link >= 0] == d[link >= 0]) and d2[4] == np.float32(0.3)
    order = np.argsort(S._to_signed(k), kind="stable")
    assert list(order[:2]) == [1, 2]  # -0.2 first, then 0.0 (rank 11, link 2) before -0.0 (rank 11, link 3)


def test_key_tensor_form_matches_numpy():
    import torch

    rng = np.random.default_rng(3)
    d = np.concatenate([np.float32([0.0, -0.0, 0.3, -1e-30, 1e-30]), rng.normal(0, 0.2, 200).astype(np.float32)])
    link = rng.integers(-1, 7, len(d)).astype(np.int32)
    voxel = np.where(link < 0, -1, rng.integers(0, 50000, len(d))).astype(np.int32)
    k_np = S._to_signed(S.pack_keys(d, link, voxel, 7, voxel_offset=123))
    k_t = S.pack_keys_tensor(torch.from_numpy(d), torch.from_numpy(link), torch.from_numpy(voxel), 7, 123)
    assert np.array_equal(k_t.numpy(), k_np)
    got = [x.numpy() for x in S.unpack_keys_tensor(k_t, 7, 0.3)]
    want = S.unpack_keys(S._from_signed(k_np), 7, 0.3)
    assert all(np.array_equal(a, b) for a, b in zip(got, want))


def test_shard_ranges_cover():
    for n in (0, 1, 7, 65536):
        for w in (1, 2, 3, 8):
            spans = [S.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _oracle_build(geom, extent, resolution, link_id=0):
    """Host stand-in for build_link_sdf (the GPU kernel is covered by the gpu tests)."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200.grids import LinkSdf

    return LinkSdf(extent, resolution, O.build_grid(geom, extent, resolution), link_id)


def _build_worker(rank, world, port, geoms, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sdfs = S.build_link_sdfs_sharded(geoms, 0.32, 0.02, build=_oracle_build)
    out.put((rank, [(s.link_id, np.asarray(s.values).copy()) for s in sdfs]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_link_sharded_build_gloo(world):
    """Link shards (config 3): every rank ends with every link's grid, identical to a local build."""
    import multiprocessing as mp

    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as SC

    chain = O.chain_from_doc(SC.ARM6G)
    geoms = [chain[i]["geometry"] for i in O.geometry_links(chain)][:5]  # 5 links over 2 / 3 ranks: uneven
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_build_worker, args=(r, world, port, geoms, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [O.build_grid(g, 0.32, 0.02) for g in geoms]
    for rank in range(world):
        got = results[rank]
        assert [i for i, _ in got] == list(range(len(geoms)))
        for (_, v), w in zip(got, want):
            assert np.array_equal(v, w)
