"""Write the scene file ``abi_demo.c`` reads (test infrastructure).

Host-side only (numpy + ctypes structs, no GPU): the chain table, link grid
descriptors with their segment bounds and the window tables come from the
package's own host recipes (``RobotModel.chain_table``,
``LinkSdf.core_radius/segment_bound``, ``WindowGeometry.host_tables``), so the
C program gets exactly what the Python facade would hand the library.
"""

from __future__ import annotations

import struct

import numpy as np

from paper_2309_12543_b200 import _native as N


def _section(f, data: bytes):
    f.write(struct.pack("<Q", len(data)))
    f.write(data)


def _arr(a, dtype) -> bytes:
    return np.ascontiguousarray(a, dtype=dtype).tobytes()


def write_scene(path, robot, sdfs, grid, window, q, points, repeat: int = 1, d_far_global=None):
    q = np.ascontiguousarray(q, dtype=np.float64)
    points = np.ascontiguousarray(points).reshape(-1, 3)
    if points.dtype not in (np.float32, np.float64):
        points = points.astype(np.float64)
    if d_far_global is None:
        d_far_global = min(s.d_far for s in sdfs)
    with open(path, "wb") as f:
        f.write(b"LSDFABI1")
        _section(f, struct.pack("<6id", robot.n_links, len(sdfs), q.shape[0], q.shape[1], len(points), repeat,
                                float(d_far_global)))
        _section(f, bytes(robot.chain_table()))
        _section(f, _arr(robot.position_limits(), np.float64))
        _section(f, bytes(grid.c_struct()))
        for s in sdfs:
            g = N.LinkGridT()
            g.dims[:] = [int(d) for d in s.dims]
            g.d_far = float(np.float32(s.d_far))
            g.extent[:] = [float(v) for v in s.extent]
            g.resolution[:] = [float(v) for v in s.resolution]
            g.core_radius = s.core_radius()
            a, u, length, lo, hi = s.segment_bound()
            g.seg_kappa_lo, g.seg_kappa_hi, g.seg_len = lo, hi, length
            g.seg_a[:] = a
            g.seg_u[:] = u
            _section(f, bytes(g))
            # x-fastest values: (nx, ny, nz) array in Fortran order
            _section(f, np.asarray(s.values, dtype=np.float32).ravel(order="F").tobytes())
        h = window.host_tables()
        w = N.WindowT()
        w.W[:] = h["W"]
        w.n_masked = h["n_masked"]
        w.e_r = h["e_r"]
        w.Wmax = h["Wmax"]
        _section(f, bytes(w))
        _section(f, _arr(h["P"], np.float64))
        _section(f, b"" if h["zrange"] is None else _arr(h["zrange"], np.int16))
        _section(f, _arr(h["mask_bits"], np.uint32))
        _section(f, _arr(h["shell_cells"], np.uint32))
        _section(f, _arr(h["shell_radius"], np.float32))
        _section(f, q.tobytes())
        _section(f, points.tobytes())


def read_result(path, C: int):
    raw = open(path, "rb").read()
    d = np.frombuffer(raw, np.float32, C, 0)
    link = np.frombuffer(raw, np.int32, C, 4 * C)
    voxel = np.frombuffer(raw, np.int32, C, 8 * C)
    flags = np.frombuffer(raw, np.int32, 2, 12 * C)
    return d, link, voxel, flags
