"""Compare the device's precomputed Grangeat node records with the oracle plan."""
import ctypes
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]
import cbn_oracle as orc  # noqa: E402
from _cases import small_setup  # noqa: E402
from paper_1605_05231_b200 import _device, _lib, pipeline as pl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
geom, voxel, spec, cfg = small_setup(n, 8)
proj = pl.Projector(geom, cfg, n, voxel, 1)
m = ctypes.c_int64(0)
lib = _lib.load()
st = ctypes.c_void_p(_device.stream_ptr())
lib.cbn_projector_grangeat_records(proj._h, None, None, ctypes.byref(m), st)
dt = np.dtype([("lu", "<i2"), ("lv", "<i2"), ("col", "<i4"), ("fac", "<f4", 2), ("w", "<f4", 10)])
rec = np.zeros(m.value, dtype=dt)
perm = np.zeros(m.value, dtype=np.int32)
lib.cbn_projector_grangeat_records(proj._h, ctypes.c_void_p(rec.ctypes.data),
                                   perm.ctypes.data_as(_lib.P_i32), ctypes.byref(m), st)
gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
print("perm is a permutation:", np.array_equal(np.sort(perm), np.arange(m.value)))
w_ref = np.concatenate([gp.plan.weights[0], gp.plan.weights[1]], 1)[perm] / orc.kb_kernel(
    0.0, 5, gp.plan.betas[0])
w_dev = rec["w"]
err = np.abs(w_dev - w_ref).max(1)
bad = np.nonzero(err > 1e-5)[0]
print("weight mismatches:", len(bad))
for k in bad[:10]:
    i = perm[k]
    print("node", i, "mu", i // cfg.n_t, "t", i % cfg.n_t, "dev", np.round(w_dev[k], 5),
          "ref", np.round(w_ref[k], 5))
print("col ok:", np.array_equal(rec["col"] // cfg.n_t, perm // cfg.n_t))
# bin origins implied by the records, and a host emulation of the binned spread
K = 2 * n
fu = np.mod(gp.plan.first[0], K).astype(int)[perm]
fv = np.mod(gp.plan.first[1], K).astype(int)[perm]
ou, ov = fu - rec["lu"], fv - rec["lv"]
print("lu/lv in [0,8):", bool(((rec["lu"] >= 0) & (rec["lu"] < 8) & (rec["lv"] >= 0) & (rec["lv"] < 8)).all()),
      "origins multiple of 8:", bool(((ou % 8) == 0).all() and ((ov % 8) == 0).all()))
rng = np.random.default_rng(3)
y = rng.standard_normal(m.value) + 1j * rng.standard_normal(m.value)   # per sorted record
grid = np.zeros((K, K), complex)
for k in range(m.value):
    for a in range(5):
        for b in range(5):
            grid[(ou[k] + rec["lu"][k] + a) % K, (ov[k] + rec["lv"][k] + b) % K] += rec["w"][k][a] * rec["w"][k][5 + b] * y[k]
ref = np.zeros((K, K), complex)
for k in range(m.value):
    i = perm[k]
    for a in range(5):
        for b in range(5):
            ref[int(gp.plan.first[0][i] + a) % K, int(gp.plan.first[1][i] + b) % K] += gp.plan.weights[0][i][a] * gp.plan.weights[1][i][b] * y[k]
ref /= orc.kb_kernel(0.0, 5, gp.plan.betas[0]) ** 2
print("host emulation vs oracle spread:", np.linalg.norm(grid - ref) / np.linalg.norm(ref))
