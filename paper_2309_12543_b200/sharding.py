"""Multi-GPU partitioning of the batched query.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.

* **Waypoint shards** (the throughput sweep, config 4): waypoints are
  independent ("partitioned by configuration is the contract"),
  so rank r runs the query on its contiguous slice and nothing crosses the
  interconnect on the data path; :func:`gather_waypoint_results` collects the
  (d, link, voxel) slices when a caller wants them in one place.
* **Obstacle shards** (huge clouds, few waypoints): each rank evaluates every
  waypoint against its slice of the sorted occupied-voxel list; the per-rank
  winners are combined with ONE min all-reduce of a packed 64-bit key
  (orderable f32 distance, global voxel rank, link) — the same lexicographic
  key the kernel reduces with, so the tie rule (lowest rank, then lowest link)
  and the clamp rule survive the reduction exactly.  C = 500 keys = 4 KB.

The key helpers are plain numpy so the reduction logic is tested on CPU
(gloo, world size 2) in tests/test_sharding.py.
"""

from __future__ import annotations

import numpy as np

_SIGN = np.uint64(1 << 63)
_NONE = np.uint64(0xFFFFFFFFFFFFFFFF)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n items for rank (the last rank takes the remainder)."""
    per = n // world
    lo = rank * per
    hi = n if rank == world - 1 else lo + per
    return lo, hi


def orderable(d: np.ndarray) -> np.ndarray:
    """f32 -> u32 preserving order, -0.0 == +0.0 (lsdf_math.cuh::orderable)."""
    d = np.asarray(d, dtype=np.float32).copy()
    d[d == 0] = 0.0
    b = d.view(np.uint32)
    return np.where(b & np.uint32(0x80000000), ~b, b | np.uint32(0x80000000)).astype(np.uint32)


def from_orderable(k: np.ndarray) -> np.ndarray:
    k = np.asarray(k, dtype=np.uint32)
    b = np.where(k & np.uint32(0x80000000), k & np.uint32(0x7FFFFFFF), ~k).astype(np.uint32)
    return b.view(np.float32)


def pack_keys(d, link, voxel, n_links: int, voxel_offset: int = 0) -> np.ndarray:
    """(d, link, voxel) of one shard -> u64 keys; -1 entries (nothing below the clamp) -> max key."""
    d = np.asarray(d, dtype=np.float32)
    link = np.asarray(link, dtype=np.int64)
    voxel = np.asarray(voxel, dtype=np.int64)
    lo = (voxel + voxel_offset) * n_links + link
    keys = (orderable(d).astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)
    return np.where(link < 0, _NONE, keys)


def unpack_keys(keys, n_links: int, clamp: float):
    keys = np.asarray(keys, dtype=np.uint64)
    none = keys == _NONE
    hi = (keys >> np.uint64(32)).astype(np.uint32)
    lo = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    d = np.where(none, np.float32(clamp), from_orderable(hi)).astype(np.float32)
    link = np.where(none, -1, lo % n_links).astype(np.int32)
    voxel = np.where(none, -1, lo // n_links).astype(np.int32)
    return d, link, voxel


def _to_signed(keys: np.ndarray) -> np.ndarray:
    """u64 order -> i64 order (torch's MIN reduction is signed)."""
    return (np.asarray(keys, dtype=np.uint64) ^ _SIGN).view(np.int64)


def _from_signed(keys: np.ndarray) -> np.ndarray:
    return np.asarray(keys, dtype=np.int64).view(np.uint64) ^ _SIGN


def allreduce_min_keys(keys: np.ndarray, group=None, device=None) -> np.ndarray:
    """Element-wise min of u64 keys over all ranks (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(_to_signed(keys).copy())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return _from_signed(t.cpu().numpy())


# ---- the same keys as torch tensors (device-resident on the NCCL path: no host round trip)

_I64_MIN = -(1 << 63)
_I64_MAX = (1 << 63) - 1


def pack_keys_tensor(d, link, voxel, n_links: int, voxel_offset: int = 0):
    """Torch form of :func:`pack_keys` in signed order (key ^ 2^63 as int64, for a MIN all-reduce).

    d f32, link / voxel int32 tensors on any device; -1 links map to the largest key.
    """
    import torch

    d = torch.where(d == 0, torch.zeros_like(d), d)  # -0.0 == +0.0
    b = d.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    neg = (b & 0x80000000) != 0
    ordr = torch.where(neg, (~b) & 0xFFFFFFFF, b | 0x80000000)
    lo = (voxel.to(torch.int64) + voxel_offset) * n_links + link.to(torch.int64)
    key = ((ordr << 32) | lo) ^ _I64_MIN  # u64 bits, flipped into signed order
    return torch.where(link < 0, torch.full_like(key, _I64_MAX), key)


def unpack_keys_tensor(keys, n_links: int, clamp: float):
    """Inverse of :func:`pack_keys_tensor` -> (d f32, link i32, voxel i32) tensors, clamp rule applied."""
    import torch

    none = keys == _I64_MAX
    u = keys ^ _I64_MIN
    hi = (u >> 32) & 0xFFFFFFFF
    lo = u & 0xFFFFFFFF
    bits = torch.where((hi & 0x80000000) != 0, hi & 0x7FFFFFFF, (~hi) & 0xFFFFFFFF)
    d = bits.to(torch.int32).view(torch.float32)  # low 32 bits reinterpret (two's complement wrap)
    d = torch.where(none, torch.full_like(d, float(np.float32(clamp))), d)
    link = torch.where(none, torch.full_like(lo, -1), lo % n_links).to(torch.int32)
    voxel = torch.where(none, torch.full_like(lo, -1), lo // n_links).to(torch.int32)
    return d, link, voxel


def query_obstacle_sharded(traj, obstacles, group=None):
    """(d, link, voxel) over the full obstacle set, each rank evaluating its voxel slice.

    ``obstacles`` is the full (replicated) ObstacleVoxelSet; rank r keeps the
    occupied voxels of rank [lo, hi) in the sorted list, queries them on its
    GPU, and the packed keys meet in one MIN all-reduce.  With NCCL the keys
    are packed, reduced and unpacked on the device; only the result leaves it.
    """
    import torch
    import torch.distributed as dist

    from .query import ObstacleVoxelSet, query_min_distances

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(obstacles.n_occupied, rank, world)
    part = ObstacleVoxelSet(indices=obstacles.indices[lo:hi], grid=obstacles.grid, n_points=obstacles.n_points,
                            n_dropped=obstacles.n_dropped, _sorted_unique=True)
    if dist.get_backend(group) == "nccl":
        C_ = traj.n_configs
        if part.n_occupied:
            occ, by_pos = part.occupancy()
            out = traj.query_device(occ, by_pos)
            keys = pack_keys_tensor(out["d"], out["link"], out["voxel"], traj.n_links, voxel_offset=lo)
        else:
            keys = torch.full((C_,), _I64_MAX, dtype=torch.int64, device=torch.cuda.current_device())
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
        d, link, voxel = unpack_keys_tensor(keys, traj.n_links, traj.d_far_global)
        return d.cpu().numpy(), link.cpu().numpy(), voxel.cpu().numpy()
    d, link, voxel = query_min_distances(traj, part, return_argmin=True)
    keys = pack_keys(d, link, voxel, traj.n_links, voxel_offset=lo)
    return unpack_keys(allreduce_min_keys(keys, group), traj.n_links, traj.d_far_global)


def gather_waypoint_results(d, link, voxel, group=None):
    """All-gather the per-rank waypoint slices (variable lengths) into full arrays on every rank.

    Inputs are numpy arrays or tensors.  With NCCL every buffer lives on this
    rank's GPU (NCCL cannot move host tensors); gloo gathers host tensors.
    Returns numpy (d f32, link i32, voxel i32) in rank order.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")

    def as_t(x, dtype):
        return (x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))).to(dev, dtype)

    d_t, l_t, v_t = as_t(d, torch.float32), as_t(link, torch.int32), as_t(voxel, torch.int32)
    n = torch.tensor([d_t.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    # one int32 block per rank: d bits, link, voxel (exact, 12 B per waypoint)
    mine = torch.zeros((m, 3), dtype=torch.int32, device=dev)
    mine[: d_t.shape[0], 0] = d_t.view(torch.int32)
    mine[: d_t.shape[0], 1] = l_t
    mine[: d_t.shape[0], 2] = v_t
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    rows = torch.cat([p[:s] for p, s in zip(parts, sizes)]).cpu()
    return (rows[:, 0].contiguous().view(torch.float32).numpy(), rows[:, 1].numpy().astype(np.int32),
            rows[:, 2].numpy().astype(np.int32))


def build_link_sdfs_sharded(geometries, extent, resolution, group=None, build=None):
    """Per-link SDF precompute partitioned by link.

    Rank r builds links r, r + world, ... (``build_link_sdf`` on its GPU by
    default), then ONE all-gather of the padded (links-per-rank, cells) f32
    block gives every rank every grid (NCCL on GPUs — 8 MiB per 128^3 link —
    gloo on CPU).  Returns the LinkSdf list in link order on every rank.
    """
    import torch
    import torch.distributed as dist

    from .grids import LinkSdf

    if build is None:
        from .meshes import build_link_sdf as build
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = len(geometries)
    per = -(-n // world)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    mine = list(range(rank, n, world))
    built = [build(geometries[i], extent, resolution, link_id=i) for i in mine]
    from .grids import _cells, _vec3  # a rank without links still needs the block shape

    dims = tuple(int(d) for d in _cells(_vec3(extent, "extent"), _vec3(resolution, "resolution"), "LinkSdf"))
    ncell = int(np.prod(dims))
    block = torch.zeros((per, ncell), dtype=torch.float32, device=dev)
    for j, sdf in enumerate(built):
        if nccl:
            block[j] = sdf.device_values()
        else:
            block[j] = torch.from_numpy(np.ascontiguousarray(np.asarray(sdf.values).ravel(order="F")))
    parts = [torch.empty_like(block) for _ in range(world)]
    dist.all_gather(parts, block, group=group)
    out = []
    for i in range(n):
        flat = parts[i % world][i // world]
        if nccl:
            out.append(LinkSdf(extent, resolution, flat.clone(), link_id=i))
        else:
            out.append(LinkSdf(extent, resolution, flat.numpy().reshape(dims, order="F"), link_id=i))
    return out
