"""The five BASELINE.json configurations as seeded synthetic inputs.

SURVEY.md 7.1 / 8(d) fix the choices the configs leave open:
* meshes are n_x*n_y*n_z cells x 6 Kuhn tetrahedra (device generator,
  bit-identical to oracle/phfem_oracle.c:or_kuhn_mesh);
* jitter and coefficients come from the counter RNG
  u = (splitmix64(seed ^ index) >> 11) * 2^-53 (seed 2509 for the jitter,
  11133 for coefficients), so CPU and GPU inputs are identical;
* configs 1 and 4 state c = 0, for which no element-local Schur complement
  exists (every A_T = K_T is singular, SURVEY finding 2): they run with the
  reference operator c = 1 on the same meshes and the same u.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import phfem as ph

SEED_JITTER = 2509
SEED_COEF = 11133

# boundary plane bits: 0:x=0 1:x=lx 2:y=0 3:y=ly 4:z=0 5:z=lz
ALL_PLANES = 0x3F


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform(seed: int, idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    return (splitmix64(np.uint64(seed) ^ idx) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def log_uniform_a(ne: int, seed: int = SEED_COEF) -> np.ndarray:
    """config 3: a_T = 10^U(-2, 2) per element."""
    return np.power(10.0, 4.0 * uniform(seed, np.arange(ne)) - 2.0)


def aniso_diag(ne: int, seed: int = SEED_COEF) -> np.ndarray:
    """config 5: diag(1,1,100) in a seeded random half, diag(100,1,1) elsewhere."""
    half = uniform(seed, np.arange(ne)) < 0.5
    return np.ascontiguousarray(np.where(half[:, None], [1.0, 1.0, 100.0], [100.0, 1.0, 1.0]))


@dataclass
class Config:
    name: str
    nx: int
    ny: int
    nz: int
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0
    jitter: float = 0.0
    dirichlet_mask: int = ALL_PLANES
    levels: int = 0                # red refinements applied after generation
    problem: int = ph.PROBLEM_SIN3
    coef: str = "none"             # none | log_uniform | aniso
    c: float = 1.0
    tol: float = 1e-10
    note: str = ""

    def mesh_args(self):
        return (self.nx, self.ny, self.nz, self.lx, self.ly, self.lz, self.jitter, SEED_JITTER, self.dirichlet_mask)

    def coefficients(self, ne: int):
        if self.coef == "log_uniform":
            return dict(a_elem=log_uniform_a(ne), a_diag=None)
        if self.coef == "aniso":
            return dict(a_elem=None, a_diag=aniso_diag(ne))
        return dict(a_elem=None, a_diag=None)

    def scaled(self, factor: int) -> "Config":
        """same config on a coarser grid (parity tests at oracle-friendly sizes)"""
        d = dict(self.__dict__)
        d.update(nx=max(1, self.nx // factor), ny=max(1, self.ny // factor), nz=max(1, self.nz // factor))
        return Config(**d)

    def build(self) -> ph.Mesh:
        m = ph.Mesh.kuhn(*self.mesh_args())
        for _ in range(self.levels):
            m.refine()
        k = self.coefficients(m.sizes()[1])
        if k["a_elem"] is not None or k["a_diag"] is not None or self.c != 1.0:
            m.set_coefficients(k["a_elem"], k["a_diag"], self.c)
        return m


CONFIGS = {
    1: Config("cfg1_cube6_L3_sin", 1, 1, 1, levels=3, problem=ph.PROBLEM_SIN3,
              note="1 cube -> 6 Kuhn, 3 red refinements, all Dirichlet; c=1 (c=0 has no local Schur)"),
    2: Config("cfg2_cube6_refine", 1, 1, 1, levels=0, problem=ph.PROBLEM_SIN3,
              note="refinement + connectivity, levels 0..7 (first level >= 2e7 tets is 7)"),
    3: Config("cfg3_kuhn64_jitter_loga", 64, 64, 64, jitter=0.2, dirichlet_mask=0x3, problem=ph.PROBLEM_EXPCOS,
              coef="log_uniform", note="jitter +-0.2h, a = 10^U(-2,2), Dirichlet x=0,1"),
    4: Config("cfg4_kuhn128_sin", 128, 128, 128, dirichlet_mask=0x10, problem=ph.PROBLEM_SIN3,
              note="12.6M tets, Dirichlet z=0; c=1 (c=0 has no local Schur)"),
    5: Config("cfg5_box8_aniso", 256, 32, 32, lx=8.0, dirichlet_mask=0x1, problem=ph.PROBLEM_POLYSIN, coef="aniso",
              note="[0,8]x[0,1]^2, diag(1,1,100)/diag(100,1,1) seeded halves, Dirichlet x=0"),
}
