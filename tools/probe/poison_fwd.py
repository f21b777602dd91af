"""Forward projector at config C on a fresh plan after filling freed device pages
with a constant: any read of an unwritten buffer changes the result."""
import sys, os, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl
from paper_1605_05231_b200.workloads import workload
w = workload(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
vol = torch.from_numpy(w.volume().astype(np.float32))
def rel(a, b): return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
def poison(val):
    free, _ = torch.cuda.mem_get_info()
    x = torch.full((int(free * 0.85) // 4,), val, dtype=torch.float32, device="cuda")
    del x
    torch.cuda.synchronize(); torch.cuda.empty_cache()
def run():
    proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, pl._FORWARD)
    a = proj.forward(vol.cuda()).cpu().numpy()
    b = proj.forward(vol.cuda()).cpu().numpy()
    del proj; gc.collect(); torch.cuda.synchronize(); torch.cuda.empty_cache()
    return a, b
a0, b0 = run()
print("clean repeat", rel(b0, a0), flush=True)
for val in (1000.0, float("nan"), -3.0):
    poison(val)
    a, b = run()
    print("poison", val, "first", rel(a, a0), "second", rel(b, a0), "nan", bool(np.isnan(a).any()), flush=True)
