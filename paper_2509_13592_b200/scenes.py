"""The five BASELINE.json workloads as seeded synthetic scenes (host-side inputs).

Seeding follows SURVEY.md section 8(d), which mirrors the reference harness
(pkg/src/bccblasso/experiments.py:212-223):
  geometry  subsample_preserving_aperture(make_ura(M1, M2), M, seed = 1729 + cfg)
  snapshot s: words = SeedSequence((1729, cfg, s)).generate_state(4)
              targets from default_rng(words[2]), noise seed words[3]
The reference benchmark itself is synthetic (no public dataset), so these scenes
are the stand-in for "the same seeded inputs" on the GPU box, where the reference
package is not available.
"""

from dataclasses import dataclass

import numpy as np

from .arrays import (
    Target,
    make_ura,
    snr_to_noise_variance,
    subsample_preserving_aperture,
    synthesize_snapshot,
)
from .errors import InvalidArgumentError

BASE_SEED = 1729


@dataclass(frozen=True)
class Workload:
    cfg: int
    solver: str          # "ista" | "fista" | "admm"
    m1: int
    m2: int
    elements: int
    l1: int
    l2: int
    batch: int
    targets: int
    amplitudes: str      # "unit" | "cn" | "loguniform20"
    snr_db: float
    tau_fraction: float
    iterations: int
    rho: float = 1.0
    separated: bool = False

    @property
    def grid_points(self) -> int:
        return self.l1 * self.l2

    @property
    def work_gpi(self) -> int:
        """Grid-point-iterations of the full job: batch * L1 * L2 * iterations."""
        return self.batch * self.l1 * self.l2 * self.iterations


# BASELINE.json "configs" (index 0..4 -> cfg 1..5); see SURVEY.md 8(d) table.
WORKLOADS = {
    1: Workload(1, "ista", 16, 16, 64, 64, 64, 1, 3, "unit", 20.0, 0.1, 500),
    2: Workload(2, "fista", 32, 32, 256, 256, 256, 64, 8, "cn", 15.0, 0.05, 1000),
    3: Workload(3, "admm", 64, 64, 1024, 512, 512, 256, 16, "loguniform20", 10.0, 0.05, 500),
    4: Workload(4, "fista", 64, 32, 512, 1024, 512, 1024, 10, "unit", 20.0, 0.05, 500),
    5: Workload(5, "fista", 128, 128, 4096, 4096, 4096, 32, 32, "cn", 20.0, 0.02, 1000,
                separated=True),
}


def workload(cfg: int) -> Workload:
    if cfg not in WORKLOADS:
        raise InvalidArgumentError(f"unknown config {cfg}")
    return WORKLOADS[cfg]


def geometry_for(w: Workload):
    return subsample_preserving_aperture(make_ura(w.m1, w.m2), w.elements, seed=BASE_SEED + w.cfg)


def _circ(a: float, b: float) -> float:
    d = abs(a - b) % 1.0
    return min(d, 1.0 - d)


def draw_targets(rng: np.random.Generator, k_range: tuple[int, int]) -> list[Target]:
    """Unit-modulus random-phase targets, harmonics uniform on [-1/2, 1/2)^2, count drawn from
    [k_range[0], k_range[1]] — the reference's draw sequence (experiments.py:185-194)."""
    count = int(rng.integers(k_range[0], k_range[1] + 1))
    f1 = rng.uniform(-0.5, 0.5, count)
    f2 = rng.uniform(-0.5, 0.5, count)
    phase = rng.uniform(0.0, 2.0 * np.pi, count)
    return [Target(float(f1[i]), float(f2[i]), complex(np.exp(1j * phase[i]))) for i in range(count)]


def draw_scene_targets(w: Workload, rng: np.random.Generator) -> list[Target]:
    k = w.targets
    if w.amplitudes == "unit":
        return draw_targets(rng, (k, k))
    if w.separated:
        # rejection sampling: every pair separated by >= 1/L1 in f1 OR >= 1/L2 in f2 (circular)
        f1s: list[float] = []
        f2s: list[float] = []
        while len(f1s) < k:
            a, b = rng.uniform(-0.5, 0.5, 2)
            if all(_circ(a, p) >= 1.0 / w.l1 or _circ(b, q) >= 1.0 / w.l2 for p, q in zip(f1s, f2s)):
                f1s.append(float(a))
                f2s.append(float(b))
        f1, f2 = np.array(f1s), np.array(f2s)
    else:
        f1 = rng.uniform(-0.5, 0.5, k)
        f2 = rng.uniform(-0.5, 0.5, k)
    if w.amplitudes == "cn":
        amp = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2.0)
    elif w.amplitudes == "loguniform20":
        mag = 10.0 ** (-rng.uniform(0.0, 1.0, k))       # 20 dB power dynamic range
        amp = mag * np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, k))
    else:
        raise InvalidArgumentError(f"unknown amplitude law {w.amplitudes!r}")
    return [Target(float(f1[i]), float(f2[i]), complex(amp[i])) for i in range(k)]


def snapshot_seeds(cfg: int, s: int) -> np.ndarray:
    return np.random.SeedSequence((BASE_SEED, cfg, s)).generate_state(4)


def make_scene(w: Workload, snapshots=None):
    """Geometry plus measurement matrix y (len(snapshots) x M, complex128) and targets."""
    geom = geometry_for(w)
    idx = range(w.batch) if snapshots is None else snapshots
    ys, tg = [], []
    for s in idx:
        words = snapshot_seeds(w.cfg, int(s))
        targets = draw_scene_targets(w, np.random.default_rng(int(words[2])))
        nv = snr_to_noise_variance(targets, w.snr_db)
        ys.append(synthesize_snapshot(geom, targets, nv, seed=int(words[3])))
        tg.append(targets)
    return geom, np.stack(ys), tg
