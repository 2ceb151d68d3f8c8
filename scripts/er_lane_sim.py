"""Lane-slot accounting of energy-resolving forward schedules on config 4 (CPU, numpy).

For a sample of 32-pixel warps it evaluates (approximately: fp64 numpy, not the kernels' rules)
each pair's mask bit and energy window and counts useful terms against the lane-slots each
schedule issues.  Analysis only; not used by the product path or the tests."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import make_config  # noqa: E402

cfg = make_config(4)
hc = 12.3984193
ny, nz, nx, ndy = cfg.ny, cfg.nz, cfg.det_nx, cfg.det_ny
yc = cfg.y_min + (np.arange(ny) + 0.5) * ((cfg.y_max - cfg.y_min) / ny)
zc = cfg.z_min + (np.arange(nz) + 0.5) * ((cfg.z_max - cfg.z_min) / nz)
xd = cfg.det_cx + ((np.arange(nx) + 0.5) - nx / 2) * cfg.det_pitch
yd = cfg.det_cy + ((np.arange(ndy) + 0.5) - ndy / 2) * cfg.det_pitch
dq = (cfg.q_max - cfg.q_min) / (cfg.nq - 1)
E = cfg.energy_kev
Q = cfg.nq
mx0 = cfg.mask_cx - 0.5 * cfg.mask_nx * cfg.mask_pitch
my0 = cfg.mask_cy - 0.5 * cfg.mask_ny * cfg.mask_pitch


def pairs(vox, pix):
    """(open, klo, khi, sigma) for voxels vox (flat) x pixels pix (flat)."""
    iy, iz = np.divmod(vox, nz)
    ix, jy = np.divmod(pix, ndy)
    y = yc[iy][:, None]; z = zc[iz][:, None]
    x_d = xd[ix][None, :]; y_d = yd[jy][None, :]
    sx, sy, sz = x_d + 0 * y, y_d - y, cfg.det_z - z
    r = np.sqrt(y * y + z * z)
    s = np.sqrt(sx * sx + sy * sy + sz * sz)
    cos = (y * sy + z * sz) / (r * s)
    sig = np.sqrt(np.clip((1 - cos) / 2, 0, 1))
    t = (cfg.mask_z - z) / (cfg.det_z - z)
    px = t * x_d
    py = y + t * (y_d - y)
    cx = np.floor((px - mx0) / cfg.mask_pitch).astype(int)
    cy = np.floor((py - my0) / cfg.mask_pitch).astype(int)
    inside = (cx >= 0) & (cx < cfg.mask_nx) & (cy >= 0) & (cy < cfg.mask_ny)
    op = np.zeros(inside.shape, bool)
    op[inside] = cfg.mask[cx[inside], cy[inside]] == 1
    u = (E[None, None, :] * sig[..., None] / hc - cfg.q_min) / dq
    inr = (u > -1) & (u < Q)
    any_ = inr.any(-1)
    klo = np.where(any_, inr.argmax(-1), cfg.ne)
    khi = np.where(any_, cfg.ne - 1 - inr[..., ::-1].argmax(-1), -1)
    op &= any_
    return op, klo, khi, sig


rng = np.random.default_rng(0)
nw = int(sys.argv[1]) if len(sys.argv) > 1 else 24
tot = dict(useful=0, lane=0, reg=0, e32=0, e16=0, e8=0, pairs=0, lsteps=0)
for _ in range(nw):
    p0 = rng.integers(0, nx * ndy // 32) * 32
    pix = np.arange(p0, p0 + 32)
    c0 = rng.integers(0, ny * nz // 32) * 32
    for cc in range(8):  # 8 consecutive chunks of 32 voxels
        vox = np.arange(c0 + 32 * cc, c0 + 32 * cc + 32) % (ny * nz)
        op, klo, khi, sig = pairs(vox, pix)  # [32 vox][32 pix]
        w = np.where(op, khi - klo + 1, 0)
        tot["useful"] += w.sum()
        tot["pairs"] += op.sum()
        # warp-uniform voxel (k_forward_reg): union over open lanes, blocks of 8
        for v in range(32):
            if op[v].any():
                lo, hi = klo[v][op[v]].min(), khi[v][op[v]].max()
                tot["reg"] += 32 * 8 * (hi // 8 - lo // 8 + 1)
        # per-lane streams (k_forward_lane)
        lists = [np.nonzero(op[:, l])[0] for l in range(32)]
        st = max(len(a) for a in lists)
        tot["lsteps"] += st
        for s in range(st):
            los = [klo[a[s], l] for l, a in enumerate(lists) if s < len(a)]
            his = [khi[a[s], l] for l, a in enumerate(lists) if s < len(a)]
            tot["lane"] += 32 * 8 * (max(his) // 8 - min(los) // 8 + 1)
        # lanes = energies, one pair per warp, aligned blocks of B
        for B, key in ((32, "e32"), (16, "e16"), (8, "e8")):
            tot[key] += (B * (np.where(op, khi // B - klo // B + 1, 0))).sum()
u = tot["useful"]
print("pairs", tot["pairs"], "useful terms", u, "terms/pair", u / tot["pairs"])
for k in ("reg", "lane", "e32", "e16", "e8"):
    print(f"{k:5s} slots {tot[k]:>12d}  useful fraction {u / tot[k]:.3f}")
