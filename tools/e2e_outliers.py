"""Diagnostic: per-call wall clock of the drop-in forward call with GC events
and a per-phase split of any slow call."""
import gc
import time
import numpy as np
import torch
from paper_1605_05231_b200 import _lib, _device, _hostio
from paper_1605_05231_b200 import pipeline as pl
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload

w = workload(2)
vol = Volume3D(w.volume().astype(np.float64), w.voxel)
geom, cfg = w.geom, w.cfg
T = time.perf_counter
events = []
def cb(phase, info):
    events.append((T(), phase, info.get("generation"), info.get("collected")))
gc.callbacks.append(cb)
marks = []
orig_upload, orig_dl = _hostio.upload, _hostio.download_blocks
def upload(*a, **k):
    t0 = T(); r = orig_upload(*a, **k); marks.append(("upload", T() - t0)); return r
def dl(*a, **k):
    t0 = T(); r = orig_dl(*a, **k); marks.append(("download", T() - t0)); return r
_hostio.upload, _hostio.download_blocks = upload, dl
orig_copy = _hostio.copy
def copy(dst, src, *a, **k):
    t0 = T(); orig_copy(dst, src, *a, **k); marks.append(("conv", T() - t0))
_hostio.copy = copy
for mode in ("plain", "frozen"):
    if mode == "frozen":
        gc.collect(); gc.freeze()
    print("mode", mode)
    for i in range(25):
        marks.clear(); n_ev = len(events)
        t0 = T()
        fr = pl.nufft_forward_project(vol, geom, cfg)
        dt = 1e3 * (T() - t0)
        del fr
        flag = " <-- slow" if dt > 16 else ""
        gcs = [(ph, g, c) for (_, ph, g, c) in events[n_ev:] if ph == "stop"]
        print(f"call {i:2d} {dt:7.2f} ms gc={gcs}{flag}")
        if flag:
            print("     ", [(n, round(1e3 * v, 2)) for n, v in marks])
