"""Batched device API over the C-ABI (torch tensors in HBM, no host copies).

These are the ``*_batched`` siblings of the reference entry points: one call
processes B independent realizations with the sm_100a kernels of
libxlmimo_b200.so.  The single-realization mirrors in linsolve.py /
precoder.py / metrics.py are thin wrappers over these.

Layouts (reference layout, batch-major, C-order): H[B, M, K], A/X[B, K, K],
W/F[B, M, K].  complex64 runs the fp32/tensor-core path, complex128 the fp64
path.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib as L
from .errors import ConfigurationError

METHODS = {"jacpcg": L.XL_JACPCG, "cg": L.XL_CG, "direct": L.XL_DIRECT}
VARIANTS = {"textbook": L.XL_TEXTBOOK, "algorithm": L.XL_ALGORITHM}
# solve_batched also runs the stationary splittings (linsolve.py:128-176)
SOLVE_METHODS = dict(METHODS, jor=L.XL_JOR, gs=L.XL_GS)


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.complex64:
        return L.XL_C64
    if dt == torch.complex128:
        return L.XL_C128
    raise ConfigurationError(f"channel dtype must be complex64 or complex128, got {dt}")


def _check_tensor(t, name, ndim, dt=None):
    if not isinstance(t, torch.Tensor):
        raise ConfigurationError(f"{name} must be a torch tensor on the GPU")
    if not t.is_cuda:
        raise ConfigurationError(f"{name} must live on a CUDA device (no CPU fallback)")
    if t.dim() != ndim:
        raise ConfigurationError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if dt is not None and t.dtype != dt:
        raise ConfigurationError(f"{name} must be {dt}, got {t.dtype}")
    if not t.is_contiguous():
        raise ConfigurationError(f"{name} must be contiguous")


class _Workspace:
    """Per-(device, stream) scratch buffer that only grows (no per-call
    cudaMalloc).  Keyed by stream so concurrent calls on different streams never
    share scratch; allocated on that stream, so the caching allocator's reuse
    after a grow is stream-ordered."""

    def __init__(self):
        self.buf = {}

    def get(self, device, nbytes: int, stream=None) -> torch.Tensor:
        dev = torch.device(device)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        key = (dev.index, s.cuda_stream)
        cur = self.buf.get(key)
        if cur is None or cur.numel() < nbytes:
            self.buf.pop(key, None)
            with torch.cuda.stream(s):
                cur = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
            self.buf[key] = cur
        return cur


_WS = _Workspace()


def _xi_args(xi, B, device):
    if isinstance(xi, torch.Tensor):
        xt = xi.to(device=device, dtype=torch.float64).reshape(-1).contiguous()
        if xt.numel() != B:
            raise ConfigurationError("per-realization xi must have B entries")
        if B and not bool((xt > 0).all()):   # precoder.py:55-56, per realization
            raise ConfigurationError("regularization xi must be positive for every realization")
        return 0.0, xt
    xi = float(xi)
    if not xi > 0:
        raise ConfigurationError(f"regularization xi must be positive, got {xi}")
    return xi, None


@dataclass
class PrecoderBatch:
    """Outputs of :func:`rzf_batched` (all device tensors)."""

    W: torch.Tensor            # [B, M, K] = beta * F
    beta: torch.Tensor         # [B] float64
    sum_se: torch.Tensor       # [B] float64
    status: torch.Tensor       # [B] int32 (0 = ok)
    gamma: torch.Tensor | None = None   # [B, K] float64
    F: torch.Tensor | None = None       # [B, M, K]
    X: torch.Tensor | None = None       # [B, K, K]
    iterations: torch.Tensor | None = None  # [B] int32 (want_trace)
    trace: torch.Tensor | None = None       # [B, T + 1] float64 (want_trace): _ls_error per iteration


def alloc_outputs(H: torch.Tensor, want_gamma=True, want_F=False, want_X=False):
    B, M, K = H.shape
    dev = H.device
    f64 = dict(dtype=torch.float64, device=dev)
    return PrecoderBatch(
        W=torch.empty_like(H), beta=torch.empty(B, **f64), sum_se=torch.empty(B, **f64),
        status=torch.empty(B, dtype=torch.int32, device=dev),
        gamma=torch.empty(B, K, **f64) if want_gamma else None,
        F=torch.empty_like(H) if want_F else None,
        X=torch.empty(B, K, K, dtype=H.dtype, device=dev) if want_X else None)


def rzf_workspace_bytes(H_shape, dtype, method="jacpcg") -> int:
    B, M, K = H_shape
    L.load_library()
    return int(L._lib.xl_rzf_workspace_bytes(dtype_code(dtype), METHODS[method], B, M, K))


def uses_tensor_cores(dtype, method, M, K) -> bool:
    return tensor_core_path(dtype, method, M, K) != "none"


def tensor_core_path(dtype, method, M, K) -> str:
    """"tcgen05" (fused / streaming tcgen05 kernels), "tcgen05+mma.sync" (the
    small-K kernel with tcgen05 Gram / W and the K x K solve on mma.sync),
    "mma.sync" (the small-K kernel entirely on the warp-level tensor cores) or
    "none" (SIMT / DMMA)."""
    L.load_library()
    code = int(L._lib.xl_rzf_uses_tensor_cores(dtype_code(dtype), METHODS[method], M, K))
    return {0: "none", 1: "tcgen05", 2: "mma.sync", 3: "tcgen05+mma.sync"}[code]


def rzf_batched(H: torch.Tensor, xi, power: float, method: str = "jacpcg", T: int = 4,
                variant: str = "textbook", sigma2: float = 1.0, *, want_gamma=True,
                want_F=False, want_X=False, out: PrecoderBatch | None = None,
                check: bool = True, stream=None, general: bool = False,
                want_trace: bool = False) -> PrecoderBatch:
    """Batched RZF precoder + SINR/SE (the hot path, one fused launch when the
    tcgen05 kernel covers the shape).

    Mirrors ``rzf_iterative`` / ``rzf_direct`` (precoder.py:73-91) followed by
    ``sinr_eq9`` (metrics.py:47-58) on one full-array block per realization.
    ``check=True`` copies the status vector to the host (one sync), re-runs
    realizations the fused kernel flagged XL_STATUS_RANGE on the general GPU
    kernels, and raises the reference exception of the first failing
    realization.  ``general=True`` forces the general (SIMT) kernels.
    ``want_trace=True`` also returns the solver telemetry of the reference's
    SolverOutcome (``iterations``, ``trace`` = residual_trace,
    linsolve.py:60-68, 89-91) through ``xl_rzf_traced`` (general kernels).
    """
    lib = L.lib()
    if method not in METHODS:
        raise ConfigurationError(f"unknown solver {method!r}; expected one of {sorted(METHODS)}")
    if variant not in VARIANTS:
        raise ConfigurationError(f"unknown PCG variant {variant!r}")
    _check_tensor(H, "H", 3)
    dc = dtype_code(H.dtype)
    B, M, K = H.shape
    xs, xt = _xi_args(xi, B, H.device)
    if out is None:
        out = alloc_outputs(H, want_gamma, want_F, want_X)
    else:
        _check_out(out, H)
    if want_trace:
        nt = 1 if method == "direct" else int(T) + 1
        if out.iterations is None:
            out.iterations = torch.empty(B, dtype=torch.int32, device=H.device)
        if out.trace is None:
            out.trace = torch.empty(B, nt, dtype=torch.float64, device=H.device)
        if tuple(out.trace.shape) != (B, nt) or out.trace.dtype != torch.float64 or \
                tuple(out.iterations.shape) != (B,) or out.iterations.dtype != torch.int32:
            raise ConfigurationError(f"out.trace must be float64 [{B}, {nt}], out.iterations int32 [{B}]")
        nbytes = int(lib.xl_rzf_general_workspace_bytes(dc, METHODS[method], B, M, K))
        ws = _WS.get(H.device, nbytes, stream)
        rc = lib.xl_rzf_traced(dc, METHODS[method], VARIANTS[variant], L.ptr(H), B, M, K, xs,
                               L.ptr(xt), float(power), int(T), float(sigma2), L.ptr(out.W),
                               L.ptr(out.F), L.ptr(out.beta), L.ptr(out.gamma), L.ptr(out.sum_se),
                               L.ptr(out.X), L.ptr(out.iterations), L.ptr(out.trace), L.ptr(out.status),
                               L.ptr(ws), ws.numel(), L.stream_ptr(stream))
        L.check(rc, "xl_rzf_traced")
        if check:
            L.raise_status(out.status.cpu().numpy(), "rzf_batched")
        return out
    if general:
        nbytes = int(lib.xl_rzf_general_workspace_bytes(dc, METHODS[method], B, M, K))
        fn = lib.xl_rzf_general
    else:
        nbytes = int(lib.xl_rzf_workspace_bytes(dc, METHODS[method], B, M, K))
        fn = lib.xl_rzf
    ws = _WS.get(H.device, nbytes, stream)
    rc = fn(dc, METHODS[method], VARIANTS[variant], L.ptr(H), B, M, K, xs,
            L.ptr(xt), float(power), int(T), float(sigma2), L.ptr(out.W),
            L.ptr(out.F), L.ptr(out.beta), L.ptr(out.gamma), L.ptr(out.sum_se),
            L.ptr(out.X), L.ptr(out.status), L.ptr(ws), ws.numel(),
            L.stream_ptr(stream))
    L.check(rc, "xl_rzf")
    if check:
        st = out.status.cpu().numpy()
        redo = (st == L.XL_STATUS_RANGE).nonzero()[0]
        if redo.size:
            _rerun_general(H, redo, xt if xt is not None else xs, power, method, T, variant, sigma2,
                           out, stream)
            st = out.status.cpu().numpy()
        L.raise_status(st, "rzf_batched")
    return out


def _check_out(out: PrecoderBatch, H: torch.Tensor):
    """Caller-provided outputs: shapes, dtypes, device and contiguity are
    checked before their raw pointers reach the kernels."""
    B, M, K = H.shape
    f64 = torch.float64
    want = {"W": ((B, M, K), H.dtype), "beta": ((B,), f64), "sum_se": ((B,), f64),
            "status": ((B,), torch.int32), "gamma": ((B, K), f64), "F": ((B, M, K), H.dtype),
            "X": ((B, K, K), H.dtype)}
    for name, (shape, dt) in want.items():
        t = getattr(out, name)
        if t is None:
            if name in ("W", "beta", "sum_se", "status"):
                raise ConfigurationError(f"out.{name} is required")
            continue
        _check_tensor(t, f"out.{name}", len(shape), dt)
        if tuple(t.shape) != shape:
            raise ConfigurationError(f"out.{name} must have shape {shape}, got {tuple(t.shape)}")
        if t.device != H.device:
            raise ConfigurationError(f"out.{name} must live on {H.device}")


def _rerun_general(H, idx, xi, power, method, T, variant, sigma2, out, stream):
    """Re-run flagged realizations on the general GPU kernels and scatter back.

    ``xi`` is the scalar or the device float64 copy made by ``_xi_args``."""
    it = torch.from_numpy(idx).to(H.device)
    xsub = xi.index_select(0, it) if isinstance(xi, torch.Tensor) else xi
    sub = rzf_batched(H.index_select(0, it).contiguous(), xsub, power, method, T, variant, sigma2,
                      want_gamma=out.gamma is not None, want_F=out.F is not None,
                      want_X=out.X is not None, check=False, stream=stream, general=True)
    for name in ("W", "beta", "sum_se", "status", "gamma", "F", "X"):
        dst = getattr(out, name)
        if dst is not None:
            dst.index_copy_(0, it, getattr(sub, name))


def gram_batched(H: torch.Tensor, xi, stream=None) -> torch.Tensor:
    """A_b = H_b^H H_b + xi_b I (precoder.py:53-61), Hermitian by construction."""
    lib = L.lib()
    _check_tensor(H, "H", 3)
    B, M, K = H.shape
    xs, xt = _xi_args(xi, B, H.device)
    A = torch.empty(B, K, K, dtype=H.dtype, device=H.device)
    L.check(lib.xl_gram(dtype_code(H.dtype), L.ptr(H), B, M, K, xs, L.ptr(xt), L.ptr(A),
                        L.stream_ptr(stream)), "xl_gram")
    return A


@dataclass
class SolveBatch:
    X: torch.Tensor
    iterations: torch.Tensor
    status: torch.Tensor
    trace: torch.Tensor | None = None
    iterates: torch.Tensor | None = None


def solve_batched(A: torch.Tensor, method: str = "jacpcg", T: int = 5, variant: str = "textbook",
                  S: torch.Tensor | None = None, w0: torch.Tensor | None = None,
                  precond: torch.Tensor | None = None, precond_identity: bool = False,
                  eps: float | None = None, trace: bool = False, iterates: bool = False,
                  check: bool = True, stream=None, omega: float = 0.5) -> SolveBatch:
    """Batched A_b X_b = S_b (S = identity when None): linsolve.py:109-294;
    method "jor" (relaxation omega) / "gs" run the stationary splittings
    (linsolve.py:128-176)."""
    lib = L.lib()
    if method not in SOLVE_METHODS:
        raise ConfigurationError(f"unknown solver {method!r}")
    if method in ("jor", "gs") and int(T) < 1:
        raise ConfigurationError(f"iteration count T must be >= 1, got {T}")
    if method == "jor" and not omega > 0:
        raise ConfigurationError(f"relaxation omega must be positive, got {omega}")
    if variant not in VARIANTS:
        raise ConfigurationError(f"unknown PCG variant {variant!r}")
    _check_tensor(A, "A", 3)
    B, K, K2 = A.shape
    if K != K2:
        raise ConfigurationError("A must be square")
    dc = dtype_code(A.dtype)
    if S is not None:
        _check_tensor(S, "S", 3, A.dtype)
        R = S.shape[2]
        if S.shape[:2] != (B, K):
            raise ConfigurationError("S shape mismatch")
    else:
        R = K
    if w0 is not None:
        _check_tensor(w0, "w0", 3, A.dtype)
        if tuple(w0.shape) != (B, K, R):
            raise ConfigurationError(f"w0 shape {tuple(w0.shape)} does not match rhs shape {(B, K, R)}")
    if precond is not None:
        precond = precond.to(device=A.device, dtype=torch.float64).contiguous()
    dev = A.device
    X = torch.empty(B, K, R, dtype=A.dtype, device=dev)
    its = torch.empty(B, dtype=torch.int32, device=dev)
    st = torch.zeros(B, dtype=torch.int32, device=dev)
    Tn = max(int(T), 1)
    tr = torch.empty(B, Tn + 1, dtype=torch.float64, device=dev) if trace else None
    itr = torch.empty(B, Tn, K, R, dtype=A.dtype, device=dev) if iterates else None
    nbytes = int(lib.xl_solve_workspace_bytes(dc, B, K, R))
    ws = _WS.get(dev, nbytes, stream)
    if method in ("jor", "gs"):
        rc = lib.xl_solve_stationary(dc, SOLVE_METHODS[method], L.ptr(A), B, K, L.ptr(S), R,
                                     L.ptr(w0), float(omega), int(T),
                                     -1.0 if eps is None else float(eps), L.ptr(X), L.ptr(its),
                                     L.ptr(tr), L.ptr(itr), L.ptr(st), L.ptr(ws), ws.numel(),
                                     L.stream_ptr(stream))
        L.check(rc, "xl_solve_stationary")
    else:
        rc = lib.xl_solve(dc, METHODS[method], VARIANTS[variant], L.ptr(A), B, K, L.ptr(S), R,
                          L.ptr(w0), L.ptr(precond), int(bool(precond_identity)), int(T),
                          -1.0 if eps is None else float(eps), L.ptr(X), L.ptr(its), L.ptr(tr),
                          L.ptr(itr), L.ptr(st), L.ptr(ws), ws.numel(), L.stream_ptr(stream))
        L.check(rc, "xl_solve")
    if check:
        L.raise_status(st.cpu().numpy(), "solve_batched")
    return SolveBatch(X, its, st, tr, itr)


def apply_precoder_batched(H: torch.Tensor, X: torch.Tensor, power: float, sigma2: float = 1.0,
                           want_F=False, check=True, stream=None) -> PrecoderBatch:
    """F = H X, power scaling and SINR/SE for a given solution X."""
    lib = L.lib()
    _check_tensor(H, "H", 3)
    _check_tensor(X, "X", 3, H.dtype)
    B, M, K = H.shape
    out = alloc_outputs(H, True, want_F, False)
    dc = dtype_code(H.dtype)
    nbytes = int(lib.xl_apply_precoder_workspace_bytes(dc, B, M, K))
    ws = _WS.get(H.device, nbytes, stream)
    L.check(lib.xl_apply_precoder(dc, L.ptr(H), L.ptr(X), B, M, K, float(power), float(sigma2),
                                  L.ptr(out.W), L.ptr(out.F), L.ptr(out.beta), L.ptr(out.gamma),
                                  L.ptr(out.sum_se), L.ptr(out.status), L.ptr(ws), ws.numel(),
                                  L.stream_ptr(stream)), "xl_apply_precoder")
    if check:
        L.raise_status(out.status.cpu().numpy(), "apply_precoder_batched")
    return out


@dataclass
class SinrBatch:
    gamma: torch.Tensor
    se: torch.Tensor
    sum_se: torch.Tensor
    coupling: torch.Tensor   # B = H^H G


def sinr_batched(H: torch.Tensor, G: torch.Tensor, sigma2: float, stream=None) -> SinrBatch:
    """Per-user SINR/SE of precoder G (metrics.py:35-58), coupling B = H^H G."""
    lib = L.lib()
    _check_tensor(H, "H", 3)
    _check_tensor(G, "G", 3, H.dtype)
    B, M, K = H.shape
    if tuple(G.shape) != (B, M, K):
        raise ConfigurationError("G must match H's shape")
    dc = dtype_code(H.dtype)
    dev = H.device
    f64 = dict(dtype=torch.float64, device=dev)
    gamma, se, s = torch.empty(B, K, **f64), torch.empty(B, K, **f64), torch.empty(B, **f64)
    coup = torch.empty(B, K, K, dtype=H.dtype, device=dev)
    nbytes = int(lib.xl_sinr_workspace_bytes(dc, B, K))
    assert nbytes <= coup.numel() * coup.element_size() + 256
    L.check(lib.xl_sinr(dc, L.ptr(H), L.ptr(G), B, M, K, float(sigma2), L.ptr(gamma), L.ptr(se),
                        L.ptr(s), L.ptr(coup), max(nbytes, coup.numel() * coup.element_size()),
                        L.stream_ptr(stream)), "xl_sinr")
    return SinrBatch(gamma, se, s, coup)


def se_partials(sum_se: torch.Tensor, chunk: int, stream=None) -> torch.Tensor:
    """{sum, sum of squares, n} per `chunk` consecutive realizations (device)."""
    lib = L.lib()
    _check_tensor(sum_se, "sum_se", 1, torch.float64)
    B = sum_se.numel()
    nc = (B + chunk - 1) // chunk
    out = torch.empty(nc, 3, dtype=torch.float64, device=sum_se.device)
    L.check(lib.xl_se_partials(L.ptr(sum_se), B, int(chunk), L.ptr(out), L.stream_ptr(stream)),
            "xl_se_partials")
    return out


def combine_se_partials(partials) -> tuple[float, float]:
    """Mean and SEM (ddof=1) from ordered chunk partials (metrics.py:61-68)."""
    import math
    s = q = n = 0.0
    for a, b, c in partials:
        s += float(a); q += float(b); n += float(c)
    if n < 1:
        raise ConfigurationError("sum_se needs at least one trial")
    mean = s / n
    if n < 2:
        return mean, 0.0
    var = max(q - n * mean * mean, 0.0) / (n - 1)
    return mean, math.sqrt(var) / math.sqrt(n)


class GraphedRzf:
    """A fixed-shape ``rzf_batched`` call captured once into a CUDA graph and
    replayed: the whole precoder chain (fused kernel, or the general path's
    kernels and library GEMMs) leaves the host in one launch, for callers whose
    host thread is the bottleneck (tools/time_graph.py: with back-to-back calls
    the GPU time dominates and replay gains nothing at cfg1-cfg3 sizes).

        g = GraphedRzf(B, M, K, torch.complex64, xi, power)
        out = g.run(H)      # copies H into the captured input, replays, returns
                            # the captured outputs (valid until the next run)
    """

    def __init__(self, B: int, M: int, K: int, dtype, xi, power: float, method: str = "jacpcg",
                 T: int = 4, variant: str = "textbook", sigma2: float = 1.0, want_gamma: bool = True,
                 device=None):
        dev = torch.device(device or "cuda")
        self.stream = torch.cuda.Stream(dev)
        self.H = torch.zeros(B, M, K, dtype=dtype, device=dev)
        self.H[:, 0, :] = 1  # a valid input for the warm-up
        self.out = alloc_outputs(self.H, want_gamma=want_gamma)
        kw = dict(method=method, T=T, variant=variant, sigma2=sigma2, out=self.out, check=False,
                  stream=self.stream)
        self._xi = xi.to(dev).contiguous() if isinstance(xi, torch.Tensor) else xi
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):   # warm-up: workspace, modules, library handles
            rzf_batched(self.H, self._xi, power, **kw)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            rzf_batched(self.H, self._xi, power, **kw)

    def run(self, H: torch.Tensor, check: bool = True) -> PrecoderBatch:
        self.H.copy_(H)
        self.graph.replay()
        if check:
            L.raise_status(self.out.status.cpu().numpy(), "GraphedRzf")
        return self.out


class HostPipeline:
    """Host-buffer front end of the hot path: H (pinned host) -> W (pinned host).

    Chunks of ``chunk`` realizations flow through three CUDA streams with
    double-buffered device staging: H2D of chunk i+1 and D2H of chunk i-1
    overlap the fused precoder on chunk i, so end-to-end throughput is bound by
    the PCIe copies, not by the kernels.  This is the call a user with numpy /
    host data makes (the reference's API takes host arrays).
    """

    def __init__(self, M: int, K: int, dtype=torch.complex64, chunk: int = 2048, device=None):
        self.device = torch.device(device or "cuda")
        self.M, self.K, self.dtype, self.chunk = M, K, dtype, chunk
        mk = lambda: torch.empty(chunk, M, K, dtype=dtype, device=self.device)  # noqa: E731
        self.Hd = [mk(), mk()]
        self.outs = [alloc_outputs(self.Hd[0], want_gamma=False) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_comp = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)

    def run(self, H_host: torch.Tensor, W_host: torch.Tensor, sum_se_host: torch.Tensor,
            status_host: torch.Tensor, xi, power, method="jacpcg", T=4, variant="textbook",
            sigma2=1.0):
        B = H_host.shape[0]
        n = (B + self.chunk - 1) // self.chunk
        xi_dev = None
        if isinstance(xi, torch.Tensor):   # per-realization xi: one device copy, sliced per chunk
            xi_dev = xi.reshape(-1).to(device=self.device, dtype=torch.float64)
            if xi_dev.numel() != B:
                raise ConfigurationError("per-realization xi must have B entries")
        ev_h = [torch.cuda.Event() for _ in range(2)]
        ev_c = [torch.cuda.Event() for _ in range(2)]
        ev_hfree = [torch.cuda.Event() for _ in range(2)]
        ev_wfree = [torch.cuda.Event() for _ in range(2)]
        started_h = [False, False]
        started_w = [False, False]
        for i in range(n):
            j = i % 2
            lo, hi = i * self.chunk, min(B, (i + 1) * self.chunk)
            nb = hi - lo
            Hd, out = self.Hd[j], self.outs[j]
            with torch.cuda.stream(self.s_h2d):
                if started_h[j]:
                    self.s_h2d.wait_event(ev_hfree[j])
                Hd[:nb].copy_(H_host[lo:hi], non_blocking=True)
                ev_h[j].record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(ev_h[j])
                if started_w[j]:
                    self.s_comp.wait_event(ev_wfree[j])
                view = out if nb == self.chunk else PrecoderBatch(
                    W=out.W[:nb], beta=out.beta[:nb], sum_se=out.sum_se[:nb],
                    status=out.status[:nb])
                xc = xi_dev[lo:hi] if xi_dev is not None else xi
                rzf_batched(Hd[:nb], xc, power, method=method, T=T, variant=variant,
                            sigma2=sigma2, want_gamma=False, out=view, check=False,
                            stream=self.s_comp)
                ev_c[j].record(self.s_comp)
                ev_hfree[j].record(self.s_comp)
                started_h[j] = True
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev_c[j])
                W_host[lo:hi].copy_(out.W[:nb], non_blocking=True)
                sum_se_host[lo:hi].copy_(out.sum_se[:nb], non_blocking=True)
                status_host[lo:hi].copy_(out.status[:nb], non_blocking=True)
                ev_wfree[j].record(self.s_d2h)
                started_w[j] = True
        self.s_d2h.synchronize()
        self.s_comp.synchronize()
        self._rerun_range(H_host, W_host, sum_se_host, status_host, xi, power, method, T, variant,
                          sigma2)

    def _rerun_range(self, H_host, W_host, sum_se_host, status_host, xi, power, method, T,
                     variant, sigma2):
        """The rzf_batched(check=True) contract on host buffers: realizations
        the fused kernel flagged XL_STATUS_RANGE are re-run on the general
        kernels and their W / sum-SE / status scattered back."""
        st = status_host[: H_host.shape[0]].numpy()
        redo = (st == L.XL_STATUS_RANGE).nonzero()[0]
        if not redo.size:
            return
        it = torch.from_numpy(redo)
        Hd = H_host.index_select(0, it).to(self.device)
        xsub = xi
        if isinstance(xi, torch.Tensor):
            xsub = xi.reshape(-1).to(torch.float64).cpu().index_select(0, it)
        sub = rzf_batched(Hd, xsub, power, method, T, variant, sigma2, want_gamma=False,
                          check=False, general=True)
        W_host.index_copy_(0, it, sub.W.cpu())
        sum_se_host.index_copy_(0, it, sub.sum_se.cpu())
        status_host.index_copy_(0, it, sub.status.cpu())
