"""The BASELINE.json configs as named presets (synthetic inputs only).

  c1  configs[0]  256 x 256 fp64, L=4, single Sigma (BASELINE values), seed 0
  c2  configs[1]  1024 x 1024 fp32, L=4, 4 quadrant Sigmas A A^H/3 + 0.1 I
  c3  configs[2]  10000 x 40000 fp32, L=4, per-row Sigma (kappa <= 1e3)   <- bench
  c4  configs[3]  10000 x 40000 fp64, L=8, per-row Sigma + 1% near-singular
  c5  configs[4]  2048 x 2048 fp32, L=4, 8 classes on a 64-px checkerboard,
                  23 x 23 window (R = 11), h = 1
  ctx_sim         the paper's simulated batch size,
                  5,469,354 matrices G G^H, G uniform, fp64
  ctx_airsar      stand-in for the 450 x 600 AIRSAR scene (
                  the data set is not available): c2's law at 450 x 600, fp64
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .wishart import sigma as _sigma

MODE_SINGLE, MODE_QUADRANT, MODE_ROW, MODE_CHECKER, MODE_PAPER_SIM = 0, 1, 2, 3, 4


@dataclass(frozen=True)
class Config:
    name: str
    height: int
    width: int
    dtype: str              # "float32" | "float64" (storage)
    looks: int
    mode: int
    seed: int = 0
    stream: int = 0
    near_singular_frac: float = 0.0
    radius: int = 0         # window configs only
    h: float = 1.0
    baseline_index: int = -1
    notes: str = field(default="", compare=False)

    @property
    def n(self) -> int:
        return self.height * self.width

    def table(self, height: int | None = None) -> np.ndarray:
        """Cholesky table (rows x 9, fp64) for this config."""
        H = self.height if height is None else height
        if self.mode == MODE_SINGLE:
            sig = _sigma.SIGMA_C1[None]
        elif self.mode == MODE_QUADRANT:
            sig = _sigma.random_hpd(4, self.seed, self.stream)
        elif self.mode == MODE_CHECKER:
            sig = _sigma.random_hpd(8, self.seed, self.stream)
        elif self.mode == MODE_ROW:
            sig = _sigma.per_row(H, self.seed, self.stream)
        else:
            return np.zeros((1, 9))
        return _sigma.cholesky_table(sig)

    def scaled(self, height: int, width: int | None = None, name: str | None = None) -> "Config":
        """Same law on another image size (tests and sampled runs)."""
        d = dict(self.__dict__)
        d["height"] = height
        d["width"] = self.width if width is None else width
        d["name"] = name or f"{self.name}@{height}x{d['width']}"
        return Config(**d)


CONFIGS = {
    "c1": Config("c1", 256, 256, "float64", 4, MODE_SINGLE, stream=1, baseline_index=0),
    "c2": Config("c2", 1024, 1024, "float32", 4, MODE_QUADRANT, stream=2, baseline_index=1),
    "c3": Config("c3", 10000, 40000, "float32", 4, MODE_ROW, stream=3, baseline_index=2),
    "c4": Config("c4", 10000, 40000, "float64", 8, MODE_ROW, stream=4, near_singular_frac=0.01,
                 baseline_index=3),
    "c5": Config("c5", 2048, 2048, "float32", 4, MODE_CHECKER, stream=5, radius=11, h=1.0,
                 baseline_index=4),
    "ctx_sim": Config("ctx_sim", 2, 2734677, "float64", 1, MODE_PAPER_SIM, stream=6),
    "ctx_airsar": Config("ctx_airsar", 450, 600, "float64", 4, MODE_QUADRANT, stream=7),
}


def get(name: str) -> Config:
    return CONFIGS[name]
