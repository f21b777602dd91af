"""The backprojector's den at config 2 (phi = 0 plane of the orbit-averaged
den, [theta][rho]) and its max, for comparison with the reference's den
(tests/golden/make_golden_den.py)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _lib
from paper_1605_05231_b200.workloads import workload
w = workload(2)
lib = _lib.load()
def buf(proj, name, dt):
    n = ctypes.c_int64()
    _lib.check(lib.cbn_projector_debug_buffer(proj._h, name.encode(), None, ctypes.byref(n), proj._s))
    out = np.empty(n.value, np.uint8)
    _lib.check(lib.cbn_projector_debug_buffer(proj._h, name.encode(), out.ctypes.data, ctypes.byref(n), proj._s))
    return out.view(dt).copy()
proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, pl._BACK)
proj.backproject(torch.zeros((w.geom.n_views, w.geom.nu, w.geom.nv), dtype=torch.float32, device="cuda"))
den = buf(proj, "den_cache", np.float32)
n_rho = 2 * int(np.ceil(1.5 * w.n / 2.0))
den = den.reshape(w.spec.n_phi, w.spec.n_theta, n_rho)
os.makedirs("gpurun_out", exist_ok=True)
np.savez(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/den_ours.npz", plane0=den[0], plane7=den[7],
         dmax=buf(proj, "den_max", np.float64))
print("saved", den.shape)
