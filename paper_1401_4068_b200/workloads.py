"""Synthetic ensembles for the BASELINE.json configs (input generation only).

The reference generates its benchmark inputs with its simulators
(/root/reference/pkg/src/ente/simulators.py).  These are restated here only so
that bench.py and the parity tests can rebuild the exact same ensembles on
a box without the reference; they are not on the accelerated path.  Outputs
are pinned bit-for-bit to the reference by tests/test_workloads.py
(hashes in tests/golden/workloads.npz).

* ``ar_pair``      <- simulate_ar_pair / table1_params / ar_coupling_schedules
                      simulators.py:182-245
* ``lorenz_pair``  <- simulate_lorenz_pair / _rk4_lorenz simulators.py:56-138
                      (RK4 vectorised over repetitions; same per-element
                      operation order, no contraction -> identical bits)
* ``CONFIGS``      <- SURVEY.md 8(d) C1..C5
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# (alpha_x, alpha_y, beta_yx, beta_xy, delta_yx, delta_xy) -- simulators.py:237-241
_TABLE1 = {
    "unidirectional": (0.75, 0.35, 0.0, -0.35, 0, 10),
    "two_step": (0.75, 0.35, 0.0, -0.35, 0, 10),
    "bidirectional": (0.475, 0.35, -0.4, -0.35, 20, 10),
}


def ar_pair(scenario: str, n_repetitions: int, n_samples: int, seed: int = 0,
            slope: float = 0.05, inflections=(1000, 2000), burn_in: int = 500,
            noise_scale: float = 1.0):
    """Coupled AR(1) pair with tanh-ramped couplings; returns (x, y) [R, N] fp64."""
    a_x, a_y, b_yx, b_xy, d_yx, d_xy = _TABLE1[scenario]
    d_yx = max(d_yx, 1)
    total = burn_in + n_samples
    t = (np.arange(total) - burn_in + 1).astype(np.float64)

    def ramp(t0):
        return 0.5 * (1.0 + np.tanh(slope * (t - t0)))

    i_xy, i_yx = inflections
    if scenario == "unidirectional":
        g_xy, g_yx = b_xy * ramp(i_xy), np.zeros_like(t)
    elif scenario == "two_step":
        g_xy, g_yx = b_xy * 0.5 * (ramp(i_xy) + ramp(i_yx)), np.zeros_like(t)
    else:
        g_xy, g_yx = b_xy * ramp(i_xy), b_yx * ramp(i_yx)

    nx = np.empty((n_repetitions, total))
    ny = np.empty((n_repetitions, total))
    for r in range(n_repetitions):
        gen = np.random.default_rng(np.random.SeedSequence((seed, r)))
        nx[r] = gen.standard_normal(total) * noise_scale
        ny[r] = gen.standard_normal(total) * noise_scale
    x = np.zeros((n_repetitions, total))
    y = np.zeros((n_repetitions, total))
    for s in range(total):
        xp = x[:, s - 1] if s >= 1 else 0.0
        yp = y[:, s - 1] if s >= 1 else 0.0
        yd = y[:, s - d_yx] if s >= d_yx else 0.0
        xd = x[:, s - d_xy] if s >= d_xy else 0.0
        x[:, s] = a_x * xp + g_yx[s] * yd + nx[:, s]
        y[:, s] = a_y * yp + g_xy[s] * xd + ny[:, s]
    return x[:, burn_in:].copy(), y[:, burn_in:].copy()


def _rk4(u, v, w, nsteps, dt, sigma, rho, beta, forcing):
    """RK4 over all repetitions at once; forcing is [R, nsteps+1] or None."""
    traj = np.empty((u.shape[0], nsteps + 1))
    traj[:, 0] = v
    zero = np.zeros_like(u)
    for s in range(nsteps):
        if forcing is None:
            f0 = f1 = fh = zero
        else:
            f0 = forcing[:, s]
            f1 = forcing[:, s + 1]
            fh = 0.5 * (f0 + f1)
        du1 = sigma * (v - u)
        dv1 = u * (rho - w) - v + f0
        dw1 = u * v - beta * w
        u2 = u + 0.5 * dt * du1
        v2 = v + 0.5 * dt * dv1
        w2 = w + 0.5 * dt * dw1
        du2 = sigma * (v2 - u2)
        dv2 = u2 * (rho - w2) - v2 + fh
        dw2 = u2 * v2 - beta * w2
        u3 = u + 0.5 * dt * du2
        v3 = v + 0.5 * dt * dv2
        w3 = w + 0.5 * dt * dw2
        du3 = sigma * (v3 - u3)
        dv3 = u3 * (rho - w3) - v3 + fh
        dw3 = u3 * v3 - beta * w3
        u4 = u + dt * du3
        v4 = v + dt * dv3
        w4 = w + dt * dw3
        du4 = sigma * (v4 - u4)
        dv4 = u4 * (rho - w4) - v4 + f1
        dw4 = u4 * v4 - beta * w4
        u = u + dt * (du1 + 2 * du2 + 2 * du3 + du4) / 6.0
        v = v + dt * (dv1 + 2 * dv2 + 2 * dv3 + dv4) / 6.0
        w = w + dt * (dw1 + 2 * dw2 + 2 * dw3 + dw4) / 6.0
        traj[:, s + 1] = v
    return traj


def lorenz_pair(delta_xy: int, n_repetitions: int, n_samples: int, gamma_schedule=lambda t: 0.0,
                sigma=10.0, rho=28.0, beta=8.0 / 3.0, integration_dt=0.01,
                sample_spacing=0.01, burn_in_steps=10000, seed=0):
    """Delay-coupled Lorenz pair (X drives Y); returns (x, y) [R, N] fp64."""
    sps = round(sample_spacing / integration_dt)
    nsteps = burn_in_steps + n_samples * sps
    lag = delta_xy * sps
    gamma = np.zeros(nsteps + 1)
    for s in range(nsteps + 1):
        ti = int(math.floor((s - burn_in_steps) / sps))
        gamma[s] = gamma_schedule(ti) if ti >= 1 else 0.0
    init = np.empty((2, n_repetitions, 3))
    for r in range(n_repetitions):
        for ch in range(2):
            gen = np.random.default_rng(np.random.SeedSequence((seed, r, ch)))
            init[ch, r] = (gen.uniform(-15, 15), gen.uniform(-20, 20), gen.uniform(10, 40))
    vx = _rk4(init[0, :, 0], init[0, :, 1], init[0, :, 2], nsteps, integration_dt,
              sigma, rho, beta, None)
    forcing = np.zeros((n_repetitions, nsteps + 1))
    if lag < nsteps + 1:
        forcing[:, lag:] = gamma[lag:] * vx[:, :nsteps + 1 - lag] ** 2
    vy = _rk4(init[1, :, 0], init[1, :, 1], init[1, :, 2], nsteps, integration_dt,
              sigma, rho, beta, forcing)
    if not (np.isfinite(vx).all() and np.isfinite(vy).all()):
        raise FloatingPointError("Lorenz integration diverged")
    rec = burn_in_steps + sps * np.arange(1, n_samples + 1)
    return vx[:, rec].copy(), vy[:, rec].copy()


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as concrete analyze_pair inputs."""

    name: str
    description: str
    spec: tuple          # (dim, delay) for both channels
    u_candidates: tuple
    window: tuple
    n_surrogates: int
    k: int = 4
    seed: int = 0
    window_starts: tuple = None  # many windows of window's width (TE per time point)
    n_pairs: int = 1             # channel pairs (pair p uses ensembles(p))

    def ensembles(self, pair: int = 0):
        return _ENSEMBLES[self.name](pair)

    def items(self, n_surrogates=None):
        """(u, perm_index[, t_lo]) chunk items of one pair: analyze_pair's order."""
        s = self.n_surrogates if n_surrogates is None else n_surrogates
        per = [(u, -1) for u in self.u_candidates] + [(u, i) for u in self.u_candidates
                                                      for i in range(s)]
        if self.window_starts is None:
            return per
        starts = np.asarray(self.window_starts, dtype=np.int32)
        arr = np.empty((len(starts) * len(per), 3), dtype=np.int32)  # window-major
        arr[:, :2] = np.tile(np.asarray(per, dtype=np.int32), (len(starts), 1))
        arr[:, 2] = np.repeat(starts, len(per))
        return arr

    @property
    def chunk_points(self) -> int:
        return 0  # filled by callers from the ensembles (R * window width)


_ENSEMBLES = {
    "C1": lambda p: ar_pair("unidirectional", 50, 3000, seed=p),
    "C2": lambda p: lorenz_pair(5, 500, 200, gamma_schedule=lambda t: 0.3, seed=p),
    "C4": lambda p: ar_pair("unidirectional", 500, 1600, seed=p),
    "C5": lambda p: ar_pair("bidirectional", 250, 1000, seed=p),
}

CONFIGS = {
    "C1": Workload("C1", "AR(1) unidirectional, 50 trials, dim=2, tau=1, u=1, k=4, "
                         "window (1101,1400), S=500", (2, 1), (1,), (1101, 1400), 500),
    "C2": Workload("C2", "coupled Lorenz, 500 trials, dim=3, tau=1, u=1..10, k=4, "
                         "window (121,180), S=200", (3, 1), tuple(range(1, 11)), (121, 180), 200),
    "C4": Workload("C4", "non-stationary AR(1): TE per time point t=501..1500 (window (t,t)), "
                         "500 trials, dim=2, u=10, S=200", (2, 1), (10,), (501, 501), 200,
                   window_starts=tuple(range(501, 1501))),
    "C5": Workload("C5", "MEG-shaped AR bidirectional: 20 channel pairs x 250 trials, dim=3, "
                         "u=5..17 step 2, window (801,890), S=500", (3, 1), tuple(range(5, 18, 2)),
                   (801, 890), 500, n_pairs=20),
}


# ---------------------------------------------------------------------------
# C3: the kNN + range-search sweep over chunk shapes
# ---------------------------------------------------------------------------
def c3_chunk(n: int, dim: int, c: int, tied: bool = False) -> np.ndarray:
    """Chunk c of the (n, dim) cell: default_rng(SeedSequence((0, n, dim, c))) normals.

    The tie variant rounds to one decimal, as the reference's criterion-6
    generator does (test_acceptance.py:219-220).
    """
    pts = np.random.default_rng(np.random.SeedSequence((0, n, dim, c))).standard_normal((n, dim))
    return np.round(pts, 1) if tied else pts


def c3_marginals(dim: int, layout: str):
    """Marginal column lists of a C3 cell.

    "te":    d_y = d_x = (dim - 1) // 2, the three KSG marginals
             (embedding.py:50-60; dim = 17 is the paper's 1 + 8 + 8)
    "bench": one marginal, the first (dim - 1) // 2 columns (bench.py:56;
             m = 8 at dim = 17, the `ente bench` default geometry)
    "knn":   no marginal (kNN distances only)
    """
    h = (dim - 1) // 2
    if layout == "te":
        if dim % 2 == 0 or dim < 3:
            raise ValueError("the te layout needs an odd dim >= 3")
        return [list(range(1, 1 + h)), list(range(0, 1 + h)), list(range(1, dim))]
    if layout == "bench":
        return [list(range(max(1, h)))]
    if layout == "knn":
        return []
    raise ValueError(f"unknown C3 layout {layout!r}")
