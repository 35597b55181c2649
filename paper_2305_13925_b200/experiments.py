"""Experiment outputs of the reference (experiments.py), fed by the batched GPU path.

The reference's experiment drivers write one UTF-8 CSV per scenario with a
fixed header (``CSV_COLUMNS``, experiments.py:23-28; values through ``_fmt``,
``.12g`` for floats, :33-36), an explicit truncation row when a generator
fails (:101-107) and a JSON manifest sidecar (config, seed, version,
timestamp, wall seconds, output; :112-124).  The writers here reproduce
those formats byte for byte; the rows come from batched device calls instead
of per-trial loops:

* ``rows_se_vs_m``   -- for every array size M of the grid, one channel batch
  of ``trials`` realizations (the BASELINE channel model with S = M / 64
  subarrays) and every method on it (paired, ``trials.se_grid_batched``),
  ergodic mean / SEM of sum-SE per method (experiments.py:73-80).
* ``rows_convergence`` -- median residual trace per method over the draws
  (telemetry.convergence_traces_batched, experiments.py:48-52).
* ``rows_flops``     -- the closed-form flop model (flops.py:35-69,
  experiments.py:39-45).

The reference's scenario geometry / configuration loader (its control plane)
is out of scope: the channel model and the grids are
arguments here.
"""

from __future__ import annotations

import csv
import datetime
import json
from time import perf_counter

import numpy as np

from . import __version__
from .errors import ConfigurationError

CSV_COLUMNS = {
    "flops": ["method", "K", "T", "init_flops", "per_iter_flops", "total_flops"],
    "convergence": ["method", "t", "median_ls_error", "trials"],
    "se_vs_m": ["M", "method", "mean_sum_se", "sem", "trials"],
    "ber": ["snr_db", "method", "ber", "bit_errors", "bits"],
}

TRUNCATION_MARKER = "__truncated__"


def _fmt(value) -> str:
    if isinstance(value, (float, np.floating)):
        return format(float(value), ".12g")
    return str(value)


def flop_model(method: str, K: int, T: int):
    """(init, per-iteration, total) flops of one K x K solve (flops.py:35-86)."""
    if K < 1 or T < 1:
        raise ConfigurationError("K and T must be >= 1")
    sweep = 8 * K ** 2 - 8 * K
    models = {
        "direct": (4 * K ** 3 + K - 1, 0),
        "gs": (4 * K ** 3 - 3 * K ** 2 + K, sweep),
        "jor": (2 * K ** 2 + K + 1, sweep),
        "cg": (0, 8 * K ** 2 + 46 * K - 6),
        "jacpcg": (4 * K ** 2 + 2 * K, 8 * K ** 2 + 46 * K - 6),
    }
    if method not in models:
        raise ConfigurationError(f"unknown method {method!r}")
    init, per = models[method]
    return init, per, init + T * per


def rows_flops(k_grid, methods, T):
    for K in k_grid:
        for m in methods:
            init, per, total = flop_model(m, K, T)
            yield [m, K, T, init, per, total]


def rows_se_vs_m(model_for_m, m_grid, methods, trials: int, T: int, snr_db: float, seed: int = 0,
                 variant: str = "textbook", dtype=None, chunk: int = 4096):
    """[M, method, mean_sum_se, sem, trials] per grid point.  ``model_for_m(M)``
    returns the ChannelModel of that array size; realizations are the global
    indices 0 .. trials-1 of seed ``seed + 1_000_003 * M`` (the reference folds
    M into the per-trial seeds the same way, experiments.py:55-60)."""
    import torch

    from . import batched as BT
    from . import trials as TR
    from .channel import generate_channels
    dtype = dtype or torch.complex64
    pts = []
    for m in methods:
        pts.append(TR.GridPoint(m, 0 if m == "direct" else int(T), float(snr_db)))
    for M in m_grid:
        model = model_for_m(M)
        if model.M != M:
            raise ConfigurationError(f"model for M = {M} has {model.M} antennas")
        sums = {p: [] for p in pts}
        for c0 in range(0, trials, chunk):
            nb = min(chunk, trials - c0)
            H = generate_channels(model, seed=seed + 1_000_003 * M, first=c0, B=nb, dtype=dtype)
            g = TR.se_grid_batched(H, pts, variant=variant)
            for p in pts:
                sums[p].append(g.sum_se[p])
        for p in pts:
            x = torch.cat(sums[p])
            parts = BT.se_partials(x, 2048).cpu().numpy()
            mean, sem = BT.combine_se_partials(parts)
            yield [M, p.method, mean, sem, trials]


def rows_convergence(H, xi, S, methods, T_max: int, omega: float = 1.0, variant: str = "textbook"):
    """[method, t, median_ls_error, trials] from batched residual traces."""
    from . import telemetry as TL
    traces = TL.convergence_traces_batched(H, xi, S, methods, T_max, omega=omega, variant=variant)
    n = H.shape[0]
    for m, tr in traces.items():
        for t, err in enumerate(TL.median_trace(tr)):
            yield [m, t, float(err), n]


def write_experiment(experiment: str, rows, out_path: str, config: dict, seed: int) -> str:
    """Write the CSV (header, formatted rows, truncation row on failure) and
    the manifest sidecar exactly as experiments.py:94-124 does."""
    if experiment not in CSV_COLUMNS:
        raise ConfigurationError(f"unknown experiment {experiment!r}")
    columns = CSV_COLUMNS[experiment]
    started = perf_counter()
    with open(out_path, "w", encoding="utf-8", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(columns)
        try:
            for row in rows:
                writer.writerow([_fmt(v) for v in row])
        except Exception as exc:
            writer.writerow([TRUNCATION_MARKER, type(exc).__name__] + [""] * (len(columns) - 2))
            fh.flush()
            raise
    elapsed = perf_counter() - started
    manifest = {
        "config": config,
        "seed": seed,
        "version": __version__,
        "timestamp": datetime.datetime.now(datetime.timezone.utc).isoformat(),
        "wall_seconds": elapsed,
        "output": out_path,
    }
    with open(out_path + ".manifest.json", "w", encoding="utf-8") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return out_path
