"""Backprojector stage times (timer pass) at config 2, repeated, with and
without the column strips."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _lib
from paper_1605_05231_b200.workloads import workload
w = workload(2)
lib = _lib.load()
fp = pl.Projector(w.geom, w.cfg, w.n, w.voxel, 1)
x = fp.forward(torch.from_numpy(w.volume()).cuda()); del fp
proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, 2)
for _ in range(3): proj.backproject(x)
torch.cuda.synchronize()
def stages(steps):
    lib.cbn_projector_set_timing(proj._h, 1)
    for _ in range(steps): proj.backproject(x)
    torch.cuda.synchronize()
    cnt = ctypes.c_int32(64); ms = (ctypes.c_double * 64)(); names = ctypes.create_string_buffer(4096)
    lib.cbn_projector_stage_times(proj._h, ms, ctypes.byref(cnt), names, 4096, 1)
    lib.cbn_projector_set_timing(proj._h, 0)
    return {nm: round(ms[i] / steps, 3) for i, nm in enumerate(names.value.decode().split(";")[:cnt.value])}
print(os.environ.get("CBN_RS_STRIPS", "1"), stages(1))
print(os.environ.get("CBN_RS_STRIPS", "1"), stages(5))
print(os.environ.get("CBN_RS_STRIPS", "1"), stages(5))
