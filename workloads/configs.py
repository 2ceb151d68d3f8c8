"""The five BASELINE.json configs made concrete.

Frame (BASELINE.json configs[0]): source at the origin, beam along +z, fan in
the x = 0 plane.  Voxel centres (0, y, z); detector plane z = det_z with rows
along x (out of fan) and columns along y; mask plane z = mask_z parallel to it.
All lengths mm, q in 1/Angstrom, E in keV.

Where BASELINE.json is silent the values are the readings of SURVEY.md §8(c)
items 3, 10, 17, 18 (restated in DESIGN.md).  Every array is drawn from
numpy's PCG64 seeded through SeedSequence(seed).spawn(3) -> (mask, phantom,
poisson) sub-streams, in fp64, and rounded to fp32 once (f); the mask is uint8.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np


@dataclasses.dataclass
class Config:
    name: str
    # object slice (voxel centres min + (i + 1/2) * (max - min) / n)
    ny: int
    nz: int
    y_min: float
    y_max: float
    z_min: float
    z_max: float
    # momentum-transfer nodes q_j = q_min + j (q_max - q_min)/(nq - 1)
    nq: int
    q_min: float
    q_max: float
    # source spectrum: ne bins over [e_lo, e_hi], Kramers with e_max
    ne: int
    e_lo: float
    e_hi: float
    e_max: float
    # secondary mask [mask_nx][mask_ny], 1 = open
    mask_nx: int
    mask_ny: int
    mask_z: float
    mask_pitch: float
    mask_cx: float
    mask_cy: float
    # detector [det_nx][det_ny]; centres c + (i + 1/2 - n/2) * pitch
    det_nx: int
    det_ny: int
    det_z: float
    det_pitch: float
    det_cx: float
    det_cy: float
    energy_resolving: int
    seed: int
    phantom: str            # "random4" (config 0) or "ellipses"
    n_ellipses: int = 0
    n_materials: int = 3
    p_open: float = 0.5
    scale: float = 1.0      # C_E

    # ---- arrays filled by make_config ----
    energy_kev: Optional[np.ndarray] = None
    phi: Optional[np.ndarray] = None
    mask: Optional[np.ndarray] = None
    f: Optional[np.ndarray] = None      # fp32 [ny][nz][nq]

    @property
    def n_vox(self) -> int:
        return self.ny * self.nz

    @property
    def n_det(self) -> int:
        return self.det_nx * self.det_ny

    @property
    def f_shape(self):
        return (self.ny, self.nz, self.nq)

    @property
    def g_shape(self):
        if self.energy_resolving:
            return (self.det_nx, self.det_ny, self.ne)
        return (self.det_nx, self.det_ny)

    def desc(self) -> dict:
        """Plain-value geometry description (what both sides consume)."""
        keys = ["ny", "nz", "y_min", "y_max", "z_min", "z_max", "nq", "q_min", "q_max",
                "ne", "mask_nx", "mask_ny", "mask_z", "mask_pitch", "mask_cx", "mask_cy",
                "det_nx", "det_ny", "det_z", "det_pitch", "det_cx", "det_cy",
                "energy_resolving", "scale"]
        d = {k: getattr(self, k) for k in keys}
        d.update(sai_n_theta=0, sai_theta_min=0.0, sai_theta_max=0.0)  # exact operator (no SAI)
        d["energy_kev"] = self.energy_kev
        d["phi"] = self.phi
        d["mask"] = self.mask
        return d


def _c(**kw) -> Config:
    return Config(**kw)


# SURVEY.md §8(d) table; italic values there are the readings restated in DESIGN.md.
CONFIGS = {
    0: dict(name="config0-tiny", ny=8, nz=8, y_min=-8.0, y_max=8.0, z_min=400.0, z_max=416.0,
            nq=16, q_min=0.05, q_max=0.45, ne=8, e_lo=30.0, e_hi=120.0, e_max=125.0,
            mask_nx=32, mask_ny=32, mask_z=800.0, mask_pitch=1.0, mask_cx=12.0, mask_cy=0.0,
            det_nx=16, det_ny=16, det_z=1000.0, det_pitch=1.5, det_cx=24.0, det_cy=0.0,
            energy_resolving=0, seed=0, phantom="random4", n_materials=3),
    1: dict(name="config1-medium", ny=64, nz=64, y_min=-40.0, y_max=40.0, z_min=350.0, z_max=550.0,
            nq=64, q_min=0.02, q_max=0.5, ne=32, e_lo=20.0, e_hi=150.0, e_max=155.0,
            mask_nx=256, mask_ny=256, mask_z=800.0, mask_pitch=0.5, mask_cx=31.6, mask_cy=0.0,
            det_nx=128, det_ny=128, det_z=1000.0, det_pitch=0.8, det_cx=63.2, det_cy=0.0,
            energy_resolving=0, seed=1, phantom="ellipses", n_ellipses=6, n_materials=5),
    2: dict(name="config2-paper-shaped", ny=128, nz=128, y_min=-51.2, y_max=51.2, z_min=350.0,
            z_max=550.0, nq=128, q_min=0.02, q_max=0.5, ne=64, e_lo=20.0, e_hi=150.0, e_max=155.0,
            mask_nx=512, mask_ny=512, mask_z=800.0, mask_pitch=0.25, mask_cx=31.6, mask_cy=0.0,
            det_nx=256, det_ny=256, det_z=1000.0, det_pitch=0.4, det_cx=63.2, det_cy=0.0,
            energy_resolving=0, seed=2, phantom="ellipses", n_ellipses=6, n_materials=5),
    # config 3 = config 1 geometry + Poisson data (poisson_data below), seed 3
    3: dict(name="config3-recon", ny=64, nz=64, y_min=-40.0, y_max=40.0, z_min=350.0, z_max=550.0,
            nq=64, q_min=0.02, q_max=0.5, ne=32, e_lo=20.0, e_hi=150.0, e_max=155.0,
            mask_nx=256, mask_ny=256, mask_z=800.0, mask_pitch=0.5, mask_cx=31.6, mask_cy=0.0,
            det_nx=128, det_ny=128, det_z=1000.0, det_pitch=0.8, det_cx=63.2, det_cy=0.0,
            energy_resolving=0, seed=1, phantom="ellipses", n_ellipses=6, n_materials=5),
    4: dict(name="config4-energy-resolving", ny=256, nz=192, y_min=-38.4, y_max=38.4, z_min=350.0,
            z_max=550.0, nq=128, q_min=0.02, q_max=0.5, ne=100, e_lo=20.0, e_hi=150.0, e_max=155.0,
            mask_nx=1024, mask_ny=512, mask_z=800.0, mask_pitch=0.2, mask_cx=44.4, mask_cy=0.0,
            det_nx=512, det_ny=256, det_z=1000.0, det_pitch=0.3, det_cx=88.8, det_cy=0.0,
            energy_resolving=1, seed=4, phantom="ellipses", n_ellipses=12, n_materials=5),
}


def kramers_spectrum(ne: int, e_lo: float, e_hi: float, e_max: float):
    """Bin centres E_k = e_lo + (k + 1/2)(e_hi - e_lo)/ne and weights
    phi_k proportional to (e_max - E_k)/E_k, normalised to sum 1 (Kramers)."""
    width = (e_hi - e_lo) / ne
    e = e_lo + (np.arange(ne, dtype=np.float64) + 0.5) * width
    phi = (e_max - e) / e
    phi = phi / phi.sum()
    return e, phi


def binary_mask(rng: np.random.Generator, nx: int, ny: int, p_open: float) -> np.ndarray:
    """i.i.d. Bernoulli(p_open) secondary mask, uint8 [nx][ny], 1 = open."""
    return (rng.random((nx, ny)) < p_open).astype(np.uint8)


def material_profiles(rng: np.random.Generator, n_mat: int, q: np.ndarray) -> np.ndarray:
    """Two-peak Gaussian momentum-transfer profiles: centres U[0.1,0.4],
    heights U[0.5,1], width (sigma) 0.02 1/Angstrom.  Returns [n_mat][nq] fp64."""
    out = np.zeros((n_mat, q.size))
    for m in range(n_mat):
        c = rng.uniform(0.1, 0.4, size=2)
        h = rng.uniform(0.5, 1.0, size=2)
        for p in range(2):
            out[m] += h[p] * np.exp(-((q - c[p]) ** 2) / (2.0 * 0.02 ** 2))
    return out


def _centres(lo: float, hi: float, n: int) -> np.ndarray:
    return lo + (np.arange(n) + 0.5) * ((hi - lo) / n)


def phantom(cfg: Config, rng: np.random.Generator) -> np.ndarray:
    """f[ny][nz][nq] fp64 >= 0 (rounded to fp32 by make_config)."""
    q = cfg.q_min + np.arange(cfg.nq) * ((cfg.q_max - cfg.q_min) / (cfg.nq - 1))
    mats = material_profiles(rng, cfg.n_materials, q)
    f = np.zeros((cfg.ny, cfg.nz, cfg.nq))
    if cfg.phantom == "random4":
        # each pixel air (0) or one of the materials, uniformly; amplitude U[0.5,1.5]
        lab = rng.integers(0, cfg.n_materials + 1, size=(cfg.ny, cfg.nz))
        amp = rng.uniform(0.5, 1.5, size=(cfg.ny, cfg.nz))
        for m in range(cfg.n_materials):
            sel = lab == m + 1
            f[sel] = amp[sel][:, None] * mats[m][None, :]
        return f
    # random ellipses, painted in order (last wins) on an air background
    yc = _centres(cfg.y_min, cfg.y_max, cfg.ny)
    zc = _centres(cfg.z_min, cfg.z_max, cfg.nz)
    Y, Z = np.meshgrid(yc, zc, indexing="ij")
    ey, ez = cfg.y_max - cfg.y_min, cfg.z_max - cfg.z_min
    for _ in range(cfg.n_ellipses):
        cy = rng.uniform(cfg.y_min + 0.1 * ey, cfg.y_max - 0.1 * ey)
        cz = rng.uniform(cfg.z_min + 0.1 * ez, cfg.z_max - 0.1 * ez)
        ay = rng.uniform(0.05, 0.25) * ey
        az = rng.uniform(0.05, 0.25) * ez
        rot = rng.uniform(0.0, np.pi)
        m = rng.integers(0, cfg.n_materials)
        amp = rng.uniform(0.5, 1.5)
        dy, dz = Y - cy, Z - cz
        u = dy * np.cos(rot) + dz * np.sin(rot)
        v = -dy * np.sin(rot) + dz * np.cos(rot)
        inside = (u / ay) ** 2 + (v / az) ** 2 <= 1.0
        f[inside] = amp * mats[m][None, :]
    return f


def make_config(i: int, **overrides) -> Config:
    """Config i with all arrays drawn from its seed (overrides for test variants)."""
    kw = dict(CONFIGS[i])
    kw.update(overrides)
    cfg = Config(**kw)
    ss = np.random.SeedSequence(cfg.seed)
    rng_mask, rng_ph, _ = [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(3)]
    cfg.energy_kev, cfg.phi = kramers_spectrum(cfg.ne, cfg.e_lo, cfg.e_hi, cfg.e_max)
    cfg.mask = binary_mask(rng_mask, cfg.mask_nx, cfg.mask_ny, cfg.p_open)
    cfg.f = phantom(cfg, rng_ph).astype(np.float32)
    return cfg


def seeded_rng(seed: int, stream: int) -> np.random.Generator:
    """Sub-stream `stream` (0 mask, 1 phantom, 2 poisson, >=3 test vectors)."""
    ss = np.random.SeedSequence(seed)
    return np.random.Generator(np.random.PCG64(ss.spawn(max(3, stream + 1))[stream]))


def poisson_data(l_true: np.ndarray, seed: int, mean_count: float = 1e4, background: float = 5.0):
    """Config 3 data: s = mean_count / mean(l_true),
    y ~ Poisson(s * l_true + background), r = background.

    `l_true` = A f_true computed by the caller's forward operator (the oracle in
    tests).  Returns (y fp32, r fp32, s)."""
    l_true = np.asarray(l_true, dtype=np.float64)
    s = mean_count / l_true.mean()
    rng = seeded_rng(seed, 2)
    y = rng.poisson(s * l_true + background).astype(np.float32)
    r = np.full(l_true.shape, background, dtype=np.float32)
    return y, r, s
