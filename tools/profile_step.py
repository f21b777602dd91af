#!/usr/bin/env python
"""Run one steady-state projector step between cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees exactly one step's kernels.

  python tools/profile_step.py [--config 2] [--direction forward|back]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--direction", choices=["forward", "back"], default="forward")
    args = ap.parse_args()
    import torch
    from paper_1605_05231_b200.pipeline import Projector
    from paper_1605_05231_b200.workloads import workload
    if args.config == 4:
        from paper_1605_05231_b200 import nufft
        from paper_1605_05231_b200.workloads import config4_inputs
        x, pts = config4_inputs(int(os.environ.get("CBN_C4_POINTS", 100_000_000)))
        if os.environ.get("CBN_C4_PRESORT") == "1":
            # diagnostic: the same points handed over in (approximate) bin order,
            # so that the plan's permutation is near the identity and values /
            # outputs are accessed almost sequentially
            import numpy as np
            K, two_pi = 512, 2.0 * np.pi
            cell = np.floor(np.mod(pts.astype(np.float64), two_pi) * (K / two_pi) - 4.0).astype(np.int64) % K
            key = ((cell[:, 0] // 8) * 64 + cell[:, 1] // 8) * 32 + cell[:, 2] // 16
            order = np.argsort(key, kind="stable")
            pts = np.ascontiguousarray(pts[order])
            print("points pre-sorted by bin", flush=True)
        plan = nufft.plan_nufft(x.shape, pts, 2.0, 8)
        xd = torch.from_numpy(x).cuda()

        def step():
            nufft.nufft_adjoint(plan, nufft.nufft_forward(plan, xd))
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print("profiled one config-4 step", flush=True)
        return
    w = workload(args.config)
    vol = torch.from_numpy(w.volume()).cuda()
    if args.direction == "forward":
        proj = Projector(w.geom, w.cfg, w.n, w.voxel, 1)
        step = lambda: proj.forward(vol)          # noqa: E731
    else:
        frames = Projector(w.geom, w.cfg, w.n, w.voxel, 1).forward(vol)
        proj = Projector(w.geom, w.cfg, w.n, w.voxel, 2)
        step = lambda: proj.backproject(frames)   # noqa: E731
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one step", flush=True)


if __name__ == "__main__":
    main()
