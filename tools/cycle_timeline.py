"""Timeline of one real-time cycle: event-record nodes around every launch of
the DistanceChecker cycle, captured into a CUDA graph like the product's, so
the offsets show launch gaps, overlap and the critical path.

    python tools/cycle_timeline.py [--workload config2] [--n 200] [--flush]
"""
import argparse
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config4"])
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--flush", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape(args.workload)
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    chk.q_dev.copy_(torch.from_numpy(S.random_configs(shape.robot, shape.n_waypoints, seed=21)).cuda())
    chk.p_dev.copy_(torch.from_numpy(bench._cloud(shape, 21)).cuda())
    C_, P, _ = chk._shape
    env = ctypes.byref(chk.grid.c_struct())
    tr = chk.traj
    names = ["start", "fk0", "fk1", "vox0", "vox1", "pre0", "pre1", "scan0", "scan1", "fin0", "fin1"]
    ev = {k: torch.cuda.Event(enable_timing=True, external=True) for k in names}
    main_s = torch.cuda.Stream()
    side, pre = torch.cuda.Stream(), torch.cuda.Stream()

    def cycle():
        m = torch.cuda.current_stream()
        ev["start"].record(m)
        side.wait_stream(m)
        with torch.cuda.stream(side):
            ev["fk0"].record(side)
            N.call(chk._fk_entry, chk._chain, robot.n_links, len(chk.sdfs), N.ptr(chk.q_dev), C_, robot.dof,
                   N.ptr(chk.limits), env, chk._W, None, None, N.ptr(chk.R_geo), N.ptr(chk.dt_geo),
                   N.ptr(chk.anchor_geo), N.ptr(chk.flags), side.cuda_stream)
            ev["fk1"].record(side)
        ev["vox0"].record(m)
        N.call("lsdf_voxelize_bitmap", N.ptr(chk.p_dev), 1, P, env, N.ptr(chk.ws), m.cuda_stream)
        ev["vox1"].record(m)
        pre.wait_stream(m)
        with torch.cuda.stream(pre):
            ev["pre0"].record(pre)
            N.call("lsdf_occupancy_prefix", env, N.ptr(chk.ws), pre.cuda_stream)
            ev["pre1"].record(pre)
        m.wait_stream(side)
        qa = (N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo), C_, tr.n_links, tr._table,
              ctypes.byref(chk._wstruct), env, N.ptr(chk.ws), chk._qflags, chk.d_far_global, N.ptr(chk.qws),
              N.ptr(chk.d_dev), N.ptr(chk.link_dev), N.ptr(chk.voxel_dev), None, m.cuda_stream)
        ev["scan0"].record(m)
        N.call("lsdf_query_scan", *qa)
        ev["scan1"].record(m)
        m.wait_stream(pre)
        ev["fin0"].record(m)
        N.call("lsdf_query_finalize", *qa)
        ev["fin1"].record(m)

    with torch.cuda.stream(main_s):
        for _ in range(3):
            cycle()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(main_s), torch.cuda.graph(g, stream=main_s):
        cycle()
    flush = bench.L2Flush(torch) if args.flush else (lambda: None)
    rows = []
    for k in range(args.n + 10):
        flush()
        torch.cuda._sleep(bench.SPIN_CYCLES)
        g.replay()
        torch.cuda.synchronize()
        if k >= 10:
            rows.append({n: ev["start"].elapsed_time(ev[n]) * 1e3 for n in names[1:]})
    med = {n: statistics.median(r[n] for r in rows) for n in names[1:]}
    print(f"{args.workload} flush={args.flush}: median offsets from the cycle start (us)")
    for a, b in (("fk0", "fk1"), ("vox0", "vox1"), ("pre0", "pre1"), ("scan0", "scan1"), ("fin0", "fin1")):
        print(f"  {a[:-1]:6s} {med[a]:7.1f} -> {med[b]:7.1f}   ({med[b] - med[a]:5.1f})")
    print(f"  cycle end {med['fin1']:7.1f}  p99 {np.percentile([r['fin1'] for r in rows], 99):7.1f}")


if __name__ == "__main__":
    main()
