"""Paired batched trial driver: every method x T x SNR point on ONE channel batch.

The reference runs, per Monte-Carlo trial, every precoding method on the same
draw (``_precoders_for_trial`` metrics.py:86-90, called by ``se_trial``
metrics.py:188-200) and sweeps the SNR in an outer loop (``ber_montecarlo``
metrics.py:93-146), with xi and the transmit power derived from the SNR
(config.py:58-72).  Here one resident batch H[B, M, K] plays the role of B
trials' draws and every grid point is one batched precoder call on it, so all
points are paired exactly like the reference's methods are.

SNR convention (DESIGN.md decision D-2): sigma2 = 1, P_tx = SNR_lin,
xi = K / SNR_lin (the reference's xi = 1 / SNR differs by the factor K, which
is a parameter, not a code path: pass ``xi_rule``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import batched as BT
from .errors import ConfigurationError


@dataclass(frozen=True)
class GridPoint:
    method: str
    T: int            # iterations (ignored by "direct"; reported as 0)
    snr_db: float


@dataclass
class SeGrid:
    """Per-point outputs of :func:`se_grid_batched` (device tensors)."""

    points: list = field(default_factory=list)
    sum_se: dict = field(default_factory=dict)    # GridPoint -> [B] float64
    beta: dict = field(default_factory=dict)      # GridPoint -> [B] float64
    status: dict = field(default_factory=dict)    # GridPoint -> [B] int32
    W: dict = field(default_factory=dict)         # GridPoint -> [B, M, K] (keep_W only)
    ms: dict = field(default_factory=dict)        # GridPoint -> device ms (timed only)

    def ergodic(self, chunk: int = 2048) -> dict:
        """Mean / SEM of sum-SE per point (sum_se, metrics.py:61-68)."""
        out = {}
        for p in self.points:
            parts = BT.se_partials(self.sum_se[p], chunk).cpu().numpy()
            out[p] = BT.combine_se_partials(parts)
        return out


def grid_points(methods=("jacpcg", "cg", "direct"), T_grid=(2, 3, 4, 5),
                snr_grid_db=(-10.0, -5.0, 0.0, 5.0, 10.0, 15.0, 20.0)) -> list:
    pts = []
    for snr in snr_grid_db:
        for m in methods:
            if m not in BT.METHODS:
                raise ConfigurationError(f"unknown solver {m!r}; expected one of {sorted(BT.METHODS)}")
            for T in ((0,) if m == "direct" else T_grid):
                if m != "direct" and int(T) < 1:
                    raise ConfigurationError(f"iteration count T must be >= 1, got {T}")
                pts.append(GridPoint(m, int(T), float(snr)))
    return pts


def default_xi(K: int, snr_db: float) -> float:
    return K / 10.0 ** (snr_db / 10.0)


_SIDE = {}


def _side_streams(device, n: int):
    """n cached side streams of a device (created once, reused by every call)."""
    key = torch.device(device).index
    lst = _SIDE.setdefault(key, [])
    while len(lst) < n:
        lst.append(torch.cuda.Stream(device=device))
    return lst[:n]


def se_grid_batched(H: torch.Tensor, points, variant: str = "textbook", sigma2: float = 1.0,
                    xi_rule=default_xi, keep_W: bool = False, timed: bool = False,
                    check: bool = True, stream=None, lanes: int = 2) -> SeGrid:
    """Run every grid point on the same batch H (paired draws).

    ``points``: GridPoints (see :func:`grid_points`).  ``timed`` records the
    device time of every point's precoder call with CUDA events on the
    stream it runs on.  ``check`` raises the reference exception of the first
    failing realization of any point (after the range re-run of rzf_batched).
    ``lanes``: the points alternate over this many streams (the calling one
    plus cached side streams, forked from and joined back into it), so a
    point's last partial wave of CTAs overlaps the next point's first.
    """
    B, M, K = H.shape
    grid = SeGrid(points=list(points))
    outs = {}
    evs = {}
    st = stream if stream is not None else torch.cuda.current_stream(H.device)
    streams = [st] + _side_streams(H.device, max(1, int(lanes)) - 1)
    shared_W = [None] * len(streams)   # one scratch W per stream (W of a point is discarded)
    fork = torch.cuda.Event()
    fork.record(st)
    for s in streams[1:]:
        s.wait_event(fork)
    for ip, p in enumerate(grid.points):
        lane = ip % len(streams)
        sp = streams[lane]
        snr_lin = 10.0 ** (p.snr_db / 10.0)
        power = sigma2 * snr_lin
        xi = xi_rule(K, p.snr_db)
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(sp)
        if keep_W or shared_W[lane] is None:
            o = BT.alloc_outputs(H, want_gamma=False)
            if not keep_W:
                shared_W[lane] = o.W
        else:
            f64 = dict(dtype=torch.float64, device=H.device)
            o = BT.PrecoderBatch(W=shared_W[lane], beta=torch.empty(B, **f64), sum_se=torch.empty(B, **f64),
                                 status=torch.empty(B, dtype=torch.int32, device=H.device))
        BT.rzf_batched(H, xi, power, method=p.method, T=max(p.T, 1), variant=variant,
                       sigma2=sigma2, out=o, check=False, stream=sp)
        if timed:
            e1.record(sp)
            evs[p] = (e0, e1)
        outs[p] = o
    for s in streams[1:]:   # join: everything after this call is ordered after every point
        j = torch.cuda.Event()
        j.record(s)
        st.wait_event(j)
    if check:
        import numpy as np
        from . import _lib as L
        for p, o in outs.items():
            s = o.status.cpu().numpy()
            redo = (s == L.XL_STATUS_RANGE).nonzero()[0]
            if redo.size:
                BT._rerun_general(H, redo, xi_rule(K, p.snr_db), sigma2 * 10.0 ** (p.snr_db / 10.0),
                                  p.method, max(p.T, 1), variant, sigma2, o, stream)
                s = o.status.cpu().numpy()
            L.raise_status(np.asarray(s), f"se_grid_batched {p}")
    for p, o in outs.items():
        grid.sum_se[p] = o.sum_se
        grid.beta[p] = o.beta
        grid.status[p] = o.status
        if keep_W:
            grid.W[p] = o.W
    if timed:
        torch.cuda.synchronize(H.device)
        grid.ms = {p: e0.elapsed_time(e1) for p, (e0, e1) in evs.items()}
    return grid
