"""The five BASELINE.json workloads as concrete (spec, PatchyConfig, SolverConfig).

Synthetic inputs with the shapes BASELINE.json names; the unspecified knobs
(coarse grids of configs 2/4/5, seeds, tolerances) are fixed here and
recorded in DESIGN.md.  Deviations from the reference's feature set
(SURVEY Appendix B): config 1 dilates the coarse target (its 26^2 coarse grid
holds no target node), configs 2/3/4/5 pass explicit target partitions,
config 4 uses a periodic heading axis and the Dubins model.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Callable, Optional

import numpy as np

from .dynamics import Dubins, ScaledSpeed, SinProduct
from .patchy import PatchyConfig
from .problems import (ControlSet, ProblemSpec, TargetSpec, discretize_circle, fibonacci_sphere,
                       partition_balls_halves, partition_octants, partition_random_directions,
                       RandomDirections,
                       partition_target, target_nodes)
from .solver import SolverConfig

SEED_C2 = 1109  # disk centres of config 2
SEED_C5 = 3577  # partition directions of config 5


@dataclass
class Workload:
    name: str
    description: str
    spec: ProblemSpec
    pcfg: PatchyConfig
    cfg: SolverConfig
    fine_shape: tuple
    coarse_shape: tuple


def _eikonal_dyn(X, a):
    X = np.atleast_2d(X)
    return np.tile(np.asarray(a, dtype=float), (X.shape[0], 1))


def c1(rule: str = "kruzkov", dtype: str = "float64", schedule: str = "async", scale: int = 1) -> Workload:
    """2D eikonal, 32 circle controls, [-2,2]^2 at 101^2, ball r=0.1, coarse
    26^2, 4 angular pieces, tol 1e-8 (CPU-runnable oracle case)."""
    n = 100 * scale + 1
    nc_ = 25 * scale + 1
    spec = ProblemSpec(name="c1-eikonal2d", dim=2, box_lo=(-2.0, -2.0), box_hi=(2.0, 2.0),
                       dynamics=_eikonal_dyn, control_set=discretize_circle(32),
                       target=TargetSpec.ball((0.0, 0.0), 0.1), model=ScaledSpeed(1.0))
    kc = 4.0 / (nc_ - 1)
    pcfg = PatchyConfig(n_patches=4, coarse_nodes=nc_, fine_nodes=n,
                        coarse_target=TargetSpec.ball((0.0, 0.0), max(0.1, kc * np.sqrt(2.0))))
    return Workload("c1", "2D eikonal 101^2, 32 controls, 4 patches", spec, pcfg,
                    SolverConfig(schedule=schedule, tol=1e-8, rule=rule, dtype=dtype), (n, n), (nc_, nc_))


def c2_centres(seed: int = SEED_C2) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-0.95, 0.95, (4, 2))


def c2(rule: str = "kruzkov", dtype: str = "float64", schedule: str = "async", n: int = 2049, nc_: Optional[int] = None,
       seed: int = SEED_C2) -> Workload:
    """2D variable speed c = 1 + 0.5 sin(2 pi x) sin(2 pi y), 64 controls,
    [-1,1]^2 at 2049^2, 4 seeded disks r=0.05 -> 8 patches, coarse 513^2."""
    nc_ = nc_ or (n - 1) // 4 + 1
    speed = SinProduct(1.0, 0.5, (2.0 * np.pi, 2.0 * np.pi))
    spec = ProblemSpec(name="c2-varspeed2d", dim=2, box_lo=(-1.0, -1.0), box_hi=(1.0, 1.0),
                       dynamics=ScaledSpeed(speed).dynamics(), control_set=discretize_circle(64),
                       target=TargetSpec.balls(c2_centres(seed), 0.05), model=ScaledSpeed(speed))
    pcfg = PatchyConfig(n_patches=8, coarse_nodes=nc_, fine_nodes=n,
                        parts=partition_balls_halves)
    return Workload("c2", f"2D variable speed {n}^2, 64 controls, 8 patches", spec, pcfg,
                    SolverConfig(schedule=schedule, tol=1e-8 if dtype == "float64" else 1e-6, rule=rule,
                                 dtype=dtype), (n, n), (nc_, nc_))


def c3(rule: str = "kruzkov", dtype: str = "float64", schedule: str = "async", n: int = 257,
       nc_: Optional[int] = None) -> Workload:
    """3D eikonal, 48 Fibonacci controls, [-1,1]^3 at 257^3, ball r=0.1 in 8
    octant pieces, coarse 65^3."""
    nc_ = nc_ or (n - 1) // 4 + 1
    spec = ProblemSpec(name="c3-eikonal3d", dim=3, box_lo=(-1.0,) * 3, box_hi=(1.0,) * 3,
                       dynamics=_eikonal_dyn, control_set=fibonacci_sphere(48),
                       target=TargetSpec.ball((0.0, 0.0, 0.0), 0.1), model=ScaledSpeed(1.0))
    pcfg = PatchyConfig(n_patches=8, coarse_nodes=nc_, fine_nodes=n, parts=partition_octants)
    return Workload("c3", f"3D eikonal {n}^3, 48 controls, 8 patches", spec, pcfg,
                    SolverConfig(schedule=schedule, tol=1e-8 if dtype == "float64" else 1e-6, rule=rule,
                                 dtype=dtype), (n,) * 3, (nc_,) * 3)


def theta_slabs(n_parts: int) -> Callable:
    def parts(target, grid, serials=None):
        # equal heading slabs by node index (robust to the 2 pi / M rounding)
        serials, _ = target_nodes(target, grid, serials)
        j = np.unravel_index(serials, grid.shape)[2]
        code = (j * n_parts) // grid.shape[2]
        return [serials[code == p] for p in range(n_parts)]
    return parts


def c4(rule: str = "kruzkov", dtype: str = "float64", schedule: str = "async", nxy: int = 257, nth: int = 128,
       cxy: Optional[int] = None, cth: Optional[int] = None) -> Workload:
    """3D Dubins (x, y, th), f = (cos th, sin th, a), a in {-1,-.5,0,.5,1},
    [-2,2]^2 x [0, 2 pi) at 257x257x128 with periodic th, target disk r=0.2
    for all th, 16 heading-slab patches, coarse 65x65x32."""
    cxy = cxy or (nxy - 1) // 4 + 1
    cth = cth or max(nth // 4, 4)
    a = np.array([[-1.0], [-0.5], [0.0], [0.5], [1.0]])
    spec = ProblemSpec(name="c4-dubins", dim=3, box_lo=(-2.0, -2.0, 0.0),
                       box_hi=(2.0, 2.0, 2.0 * np.pi), dynamics=Dubins().dynamics(),
                       control_set=ControlSet(a, "explicit-list"),
                       target=TargetSpec.ball((0.0, 0.0), 0.2), model=Dubins(),
                       periodic=(False, False, True))
    pcfg = PatchyConfig(n_patches=16, coarse_nodes=(cxy, cxy, cth), fine_nodes=(nxy, nxy, nth),
                        parts=theta_slabs(16))
    return Workload("c4", f"3D Dubins {nxy}x{nxy}x{nth}, 5 controls, 16 patches", spec, pcfg,
                    SolverConfig(schedule=schedule, tol=1e-8 if dtype == "float64" else 1e-6,
                                 rule=rule, dtype=dtype,
                                 # 4 block-local relaxations: measured best here (63 vs 70 ms)
                                 inner_sweeps=4 if schedule == "async" else None),
                    (nxy, nxy, nth), (cxy, cxy, cth))


def c5(rule: str = "kruzkov", dtype: str = "float32", schedule: str = "async", n: int = 513,
       nc_: Optional[int] = None, seed: int = SEED_C5) -> Workload:
    """3D variable speed c = 1 + 0.3 sin(pi x) sin(pi y) sin(pi z), 96
    Fibonacci controls, [-1,1]^3 at 513^3, ball r=0.15 split into 32 seeded
    random-direction pieces, coarse 129^3 (fp32 patch solves: async 0.81 s,
    Jacobi 0.89 s)."""
    nc_ = nc_ or (n - 1) // 4 + 1
    speed = SinProduct(1.0, 0.3, (np.pi, np.pi, np.pi))
    spec = ProblemSpec(name="c5-varspeed3d", dim=3, box_lo=(-1.0,) * 3, box_hi=(1.0,) * 3,
                       dynamics=ScaledSpeed(speed).dynamics(), control_set=fibonacci_sphere(96),
                       target=TargetSpec.ball((0.0, 0.0, 0.0), 0.15), model=ScaledSpeed(speed))
    pcfg = PatchyConfig(n_patches=32, coarse_nodes=nc_, fine_nodes=n,
                        parts=RandomDirections(32, seed))
    return Workload("c5", f"3D variable speed {n}^3, 96 controls, 32 patches", spec, pcfg,
                    SolverConfig(schedule=schedule, tol=1e-8 if dtype == "float64" else 1e-6, rule=rule,
                                 dtype=dtype), (n,) * 3, (nc_,) * 3)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
