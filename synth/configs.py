"""BASELINE.json configs C1..C5 as concrete synthetic recipes.

| id | atoms | lattice | r_c | model (layers, lmax) | run |
|----|-------|---------|-----|----------------------|-----|
| C1 | 16 | fcc 1^3 (L = 5.371 A < 2 r_c: multi-image) | 5.0 | (2, 1) | 1 eval + 10 NVE steps |
| C2 | 1,024 | fcc 4^3 | 6.0 | (2, 2) | 1,000 NVE steps |
| C3 | 110,592 | bcc 24^3 | 6.0 | (3, 2) = paper's l=2 model | throughput + roofline |
| C4 | 884,736 | bcc 48^3 | 6.0 | (3, 1) = paper's l=1 model | strong scaling |
| C5 | 500,000 per GPU | sc 50^3 per GPU, replicated | 6.0 | (3, 1) | weak scaling (bench) |
| CP | 6,912 per GPU | sc 12^3 per GPU, replicated | 6.0 | (3, 1) | context: the paper's granularity |

r_c = 6.0 A is Table 5's r_max (§4.5); C1's 5 A is BASELINE.json's.
"""
from __future__ import annotations

import dataclasses
import os
import tempfile

from . import nh3, weights


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    lattice: str
    cells: tuple
    r_cut: float
    n_layers: int
    lmax: int
    description: str

    @property
    def n_atoms(self) -> int:
        cx, cy, cz = self.cells
        return 4 * len(nh3.LATTICE_SITES[self.lattice]) * cx * cy * cz


CONFIGS = {
    "C1": Config("C1", "fcc", (1, 1, 1), 5.0, 2, 1, "16-atom periodic box (4 NH3), 2-layer lmax=1, r_c=5"),
    "C2": Config("C2", "fcc", (4, 4, 4), 6.0, 2, 2, "liquid NH3 1,024 atoms, 2-layer lmax=2"),
    "C3": Config("C3", "bcc", (24, 24, 24), 6.0, 3, 2, "liquid NH3 110,592 atoms, 3-layer lmax=2"),
    "C4": Config("C4", "bcc", (48, 48, 48), 6.0, 3, 1, "liquid NH3 884,736 atoms, 3-layer lmax=1"),
    "C5": Config("C5", "sc", (50, 50, 50), 6.0, 3, 1, "liquid NH3 500,000 atoms per GPU, 3-layer lmax=1"),
    # SURVEY.md §8(d) optional context row: the paper's granularity, 6,912 atoms per GPU
    "CP": Config("CP", "sc", (12, 12, 12), 6.0, 3, 1, "liquid NH3 6,912 atoms per GPU (the paper's weak-scaling size)"),
}


def system(cfg: Config | str, temperature: float = 200.0, reps=(1, 1, 1), seed: int = 0) -> nh3.System:
    """seed 0 = the recipe's default streams (orientations 1, velocities 2); seed k uses
    1 + 2k and 2 + 2k (independent instances, e.g. the >= 10 time-to-failure runs per N)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    s = nh3.maxwell_boltzmann(nh3.nh3_box(cfg.lattice, cfg.cells, structure_seed=1 + 2 * seed), temperature,
                              velocity_seed=2 + 2 * seed)
    if tuple(reps) != (1, 1, 1):
        s = nh3.replicate(s, reps)
    return s


def weight_file(cfg: Config | str, directory: str | None = None, seed: int = 0, sigma=None) -> str:
    """Path of the (cached) weight file of ``cfg``'s model at its r_c."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if directory is None:
        directory = os.path.join(tempfile.gettempdir(), "allegro_b200_weights")
    os.makedirs(directory, exist_ok=True)
    tag = "cal" if sigma is None else f"sig{sigma:g}"
    path = os.path.join(directory, f"{weights.model_key(cfg.n_layers, cfg.lmax, cfg.r_cut, seed)}_{tag}.algw")
    tmp = f"{path}.{os.getpid()}.tmp"  # per process: ranks may write concurrently
    weights.make_weight_file(tmp, cfg.n_layers, cfg.lmax, cfg.r_cut, seed, sigma)
    os.replace(tmp, path)
    return path
