"""GPU tests of the fused tcgen05 precoder kernel (complex64, K in {16, 32, 64}).

Every case is checked against the CPU oracle (complex128) on the same H,
with the north_star tolerances written here: W relative Frobenius <= 1e-4,
sum-SE relative <= 1e-4 (the kernel reaches ~2e-6 / ~1e-6).
"""

import numpy as np
import pytest
import torch

from oracle import xlmimo_oracle as O

pytestmark = pytest.mark.gpu

import paper_2305_13925_b200 as X  # noqa: E402
from paper_2305_13925_b200 import _lib as L  # noqa: E402
from paper_2305_13925_b200 import batched as BT  # noqa: E402
from paper_2305_13925_b200.errors import DegenerateChannelError  # noqa: E402

W_TOL = 1e-4
SE_TOL = 1e-4


from fp32_ref import _fp32_run, _fp32_sensitivity  # noqa: E402,F401


def relf(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _check(H, out, alpha, power, method, T, variant):
    Hn = H.cpu().numpy().astype(np.complex128)
    W = out.W.cpu().numpy()
    S = out.sum_se.cpu().numpy()
    beta = out.beta.cpu().numpy()
    gam = out.gamma.cpu().numpy() if out.gamma is not None else None
    for b in range(H.shape[0]):
        G, be, g, s = O.precoder_and_se(Hn[b], alpha, power, 1.0, method, T, variant)
        wt, st = W_TOL, SE_TOL
        if variant == "algorithm" or method == "cg":
            # the diverging Algorithm-1 recurrence amplifies round-off
            # chaotically: two fp32-level executions differ by up to ~30x the
            # distance of one of them from the complex128 oracle
            fac = 30 if variant == "algorithm" else 10
            ws, ss = _fp32_sensitivity(Hn[b], alpha, power, method, T, variant)
            wt, st = max(W_TOL, fac * ws), max(SE_TOL, fac * ss)
        assert relf(W[b], G) <= wt, (b, relf(W[b], G), wt)
        assert abs(S[b] - s) <= st * abs(s), (b, S[b], s, st)
        if variant == "algorithm":
            continue
        assert abs(beta[b] - be) <= max(1e-4, wt) * be
        if gam is not None:
            # per-user SINR: a ratio whose interference sum amplifies W's relative
            # error ~10x; for the chaotic recurrences (CG at T = 6) up to ~30x (measured)
            gfac = 30 if method == "cg" else 10
            np.testing.assert_allclose(gam[b], g, rtol=max(1e-3, gfac * wt), atol=1e-6 * np.abs(g).max())


@pytest.fixture(params=["small-k", "small-k-mma", "tcgen05"])
def small_k_path(request, monkeypatch):
    """K <= 32 shapes run on every fused kernel: the small-K kernel (default
    when M K <= 8192; at K = 32, M % 128 == 0 its Gram / W on tcgen05), the
    same with mma.sync Gram / W (XL_SMALL_K_TC=0) and the tcgen05 fused
    kernel (XL_SMALL_K_MMA=0)."""
    monkeypatch.delenv("XL_SMALL_K_MMA", raising=False)
    monkeypatch.delenv("XL_SMALL_K_TC", raising=False)
    if request.param == "tcgen05":
        monkeypatch.setenv("XL_SMALL_K_MMA", "0")
    elif request.param == "small-k-mma":
        monkeypatch.setenv("XL_SMALL_K_TC", "0")
    return request.param


def _expected_path(param, M, K):
    if K > 32 or M * K > 8192 or param == "tcgen05":
        return "tcgen05"
    if param == "small-k" and K == 32 and M % 128 == 0:
        return "tcgen05+mma.sync"
    return "mma.sync"


@pytest.mark.parametrize("S,K", [(16, 64), (4, 32), (4, 16), (2, 64), (1, 16), (64, 64), (48, 32), (8, 16),
                                 (2, 32), (3, 32)])
def test_fused_shapes_vs_oracle(S, K, small_k_path):
    assert BT.tensor_core_path(torch.complex64, "jacpcg", 64 * S, K) == _expected_path(small_k_path, 64 * S, K)
    m = X.ChannelModel(S=S, K=K, p=0.6, r=0.7)
    H = X.generate_channels(m, seed=21, first=5, B=5, dtype=torch.complex64)
    alpha, power = K / 10.0, 10.0
    out = BT.rzf_batched(H, alpha, power, T=4)
    _check(H, out, alpha, power, "jacpcg", 4, "textbook")


@pytest.mark.parametrize("method,variant", [("cg", "textbook"), ("jacpcg", "algorithm")])
@pytest.mark.parametrize("T", [1, 3, 6])
def test_fused_methods(method, variant, T, small_k_path):
    m = X.ChannelModel(S=4, K=32, p=0.5, r=0.5)
    H = X.generate_channels(m, seed=3, first=0, B=4, dtype=torch.complex64)
    out = BT.rzf_batched(H, 3.2, 10.0, method=method, T=T, variant=variant)
    _check(H, out, 3.2, 10.0, method, T, variant)


@pytest.mark.parametrize("S,K", [(1, 16), (2, 32), (3, 32), (4, 16)])
@pytest.mark.parametrize("xi_per_b", [False, True])
def test_small_k_direct_vs_oracle(S, K, xi_per_b, monkeypatch):
    """Direct RZF (precoder.py:73-78) in the small-K kernel: Gauss-Jordan on the
    warp-pair layout, against the oracle's Cholesky solve; scalar and
    per-realization xi; tcgen05 (M % 128 == 0) and mma.sync Gram / W."""
    monkeypatch.delenv("XL_SMALL_K_MMA", raising=False)
    m = X.ChannelModel(S=S, K=K, p=0.6, r=0.5)
    H = X.generate_channels(m, seed=17, first=3, B=4, dtype=torch.complex64)
    assert BT.tensor_core_path(torch.complex64, "direct", 64 * S, K) in ("mma.sync", "tcgen05+mma.sync")
    if xi_per_b:
        xi = torch.tensor([K / 10.0, K / 1.0, K / 100.0, K / 3.0], dtype=torch.float64, device="cuda")
        out = BT.rzf_batched(H, xi, 10.0, method="direct")
        Hn = H.cpu().numpy().astype(np.complex128)
        for b in range(4):
            G, _, _, s = O.precoder_and_se(Hn[b], float(xi[b]), 10.0, 1.0, "direct", 1, "textbook")
            assert relf(out.W[b].cpu().numpy(), G) <= W_TOL
            assert abs(out.sum_se[b].item() - s) <= SE_TOL * abs(s)
    else:
        out = BT.rzf_batched(H, K / 10.0, 10.0, method="direct")
        _check(H, out, K / 10.0, 10.0, "direct", 1, "textbook")


def test_fused_snr_sweep_per_realization_xi():
    """configs[1]-style SNR sweep in one batch via per-realization xi."""
    m = X.ChannelModel(S=4, K=32, p=0.5, r=0.5)
    snrs = np.array([-10.0, -5.0, 0.0, 5.0, 10.0, 15.0, 20.0])
    Hone = X.generate_channels(m, seed=9, first=0, B=1, dtype=torch.complex64)
    H = Hone.repeat(len(snrs), 1, 1).contiguous()
    xi = torch.tensor(32.0 / 10 ** (snrs / 10), dtype=torch.float64, device="cuda")
    out = BT.rzf_batched(H, xi, 1.0, T=4)
    Hn = Hone[0].cpu().numpy().astype(np.complex128)
    for i, a in enumerate(xi.cpu().numpy()):
        G, _, _, s = O.precoder_and_se(Hn, a, 1.0, 1.0, "jacpcg", 4, "textbook")
        assert relf(out.W[i].cpu().numpy(), G) <= W_TOL
        assert abs(out.sum_se[i].item() - s) <= SE_TOL * s


def test_fused_matches_general_path_and_debug_gram():
    wl = X.CONFIGS["cfg3"]
    H = X.generate_channels(wl.model, seed=2, first=0, B=6, dtype=torch.complex64)
    lib = L.lib()
    A = torch.zeros(6, wl.K, wl.K, dtype=torch.complex64, device="cuda")
    lib.xl_debug_set_gram_out(A.data_ptr())
    try:
        f = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T, want_X=True, want_F=True)
        torch.cuda.synchronize()
    finally:
        lib.xl_debug_set_gram_out(None)
    g = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T, want_X=True, want_F=True, general=True)
    Ag = BT.gram_batched(H, wl.alpha())
    assert relf(A.cpu().numpy(), Ag.cpu().numpy()) < 1e-5
    assert relf(f.X.cpu().numpy(), g.X.cpu().numpy()) < 1e-5
    assert relf(f.W.cpu().numpy(), g.W.cpu().numpy()) < 1e-5
    # F = G / beta (precoder.py:70)
    np.testing.assert_allclose(f.W.cpu().numpy(), f.F.cpu().numpy() * f.beta.cpu().numpy()[:, None, None],
                               rtol=1e-5, atol=1e-7)
    assert torch.allclose(f.sum_se, g.sum_se, rtol=1e-5)


def test_fused_degenerate_and_zero_subarrays():
    m = X.ChannelModel(S=4, K=16, p=0.3, r=0.5)
    H = X.generate_channels(m, seed=4, first=0, B=4, dtype=torch.complex64)
    H[2] = 0
    H[1, :128] = 0  # leading all-zero chunks: the fp16 scale comes from a later chunk
    out = BT.rzf_batched(H, 1.6, 10.0, T=4, check=False)
    st = out.status.cpu().tolist()
    assert st[2] == 3 and st[0] == 0 and st[1] == 0 and st[3] == 0
    with pytest.raises(DegenerateChannelError):
        BT.rzf_batched(H, 1.6, 10.0, T=4)
    keep = [0, 1, 3]
    sub = H[keep].contiguous()
    _check(sub, BT.rzf_batched(sub, 1.6, 10.0, T=4), 1.6, 10.0, "jacpcg", 4, "textbook")


@pytest.mark.parametrize("scale", [1e-6, 1e6])
def test_fused_scale_invariance(scale):
    """Power-of-two pre-scaling: W is invariant to scaling H by c with xi by c^2."""
    m = X.ChannelModel(S=4, K=32, p=0.5, r=0.5)
    H = X.generate_channels(m, seed=8, first=0, B=3, dtype=torch.complex64)
    base = BT.rzf_batched(H, 3.2, 10.0, T=4)
    Hs = (H * scale).contiguous()
    out = BT.rzf_batched(Hs, 3.2 * scale * scale, 10.0, T=4)
    # W(cH, c^2 xi) = W(H, xi) exactly (beta absorbs c); SE is not invariant
    # (sigma^2 stays fixed), so it is checked against the oracle instead
    assert relf(out.W.cpu().numpy(), base.W.cpu().numpy()) < 1e-5
    _check(Hs, out, 3.2 * scale * scale, 10.0, "jacpcg", 4, "textbook")


def test_fused_range_fallback(monkeypatch):
    """A chunk far above the first chunk's scale overflows the tcgen05
    kernel's fp16 split: it flags XL_STATUS_RANGE and rzf_batched re-runs it
    on the general kernels (check=True), matching the oracle.  The mma.sync
    small-K kernel scales every user column separately and needs no re-run."""
    m = X.ChannelModel(S=4, K=16, p=1.0, r=0.5)
    H = X.generate_channels(m, seed=5, first=0, B=2, dtype=torch.complex64)
    H[0, 192:] *= 1e4
    small = BT.rzf_batched(H, 1.6, 10.0, T=4, check=False)
    assert small.status.cpu().tolist() == [0, 0]
    _check(H, small, 1.6, 10.0, "jacpcg", 4, "textbook")
    monkeypatch.setenv("XL_SMALL_K_MMA", "0")
    raw = BT.rzf_batched(H, 1.6, 10.0, T=4, check=False)
    assert raw.status.cpu().tolist()[0] == L.XL_STATUS_RANGE
    out = BT.rzf_batched(H, 1.6, 10.0, T=4)
    assert out.status.cpu().tolist() == [0, 0]
    _check(H, out, 1.6, 10.0, "jacpcg", 4, "textbook")


@pytest.mark.parametrize("B", [1, 147, 149, 297])
def test_fused_odd_batch_sizes(B):
    """Dynamic realization claiming at batch sizes around the grid (148 CTAs)."""
    m = X.ChannelModel(S=4, K=64, p=0.5, r=0.5)
    H = X.generate_channels(m, seed=8, first=11, B=B, dtype=torch.complex64)
    out = BT.rzf_batched(H, 6.4, 10.0, T=4)
    assert (out.status == 0).all()
    idx = sorted({0, B // 2, B - 1})
    sub = BT.rzf_batched(H[idx].contiguous(), 6.4, 10.0, T=4)
    assert torch.equal(sub.W, out.W[idx]) and torch.equal(sub.sum_se, out.sum_se[idx])
    Hn = H[idx].cpu().numpy().astype(np.complex128)
    for i, b in enumerate(idx):
        G, _, _, s = O.precoder_and_se(Hn[i], 6.4, 10.0, 1.0, "jacpcg", 4, "textbook")
        assert relf(out.W[b].cpu().numpy(), G) <= 1e-4
        assert abs(out.sum_se[b].item() - s) <= 1e-4 * abs(s)


def test_fused_determinism_and_batch_independence():
    wl = X.CONFIGS["cfg3"]
    H = X.generate_channels(wl.model, seed=1, first=0, B=300, dtype=torch.complex64)
    a = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T)
    b = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T)
    assert torch.equal(a.W, b.W) and torch.equal(a.sum_se, b.sum_se)
    sub = BT.rzf_batched(H[37:41].contiguous(), wl.alpha(), wl.power(), T=wl.T)
    assert torch.equal(sub.W, a.W[37:41]) and torch.equal(sub.sum_se, a.sum_se[37:41])


@pytest.mark.parametrize("method", ["jacpcg", "cg", "direct"])
def test_small_k_determinism_and_batch_independence(method, small_k_path):
    """The small-K kernel (warp-pair named barriers, tcgen05 mbarrier, TMEM) and
    its variants: bit-identical re-runs and sub-batches (a race in an exchange
    slot or a TMEM / smem reuse would show up here; compute-sanitizer is closed
    on this pool, profiles/r02_sanitizer.md)."""
    wl = X.CONFIGS["cfg2"]
    H = X.generate_channels(wl.model, seed=4, first=0, B=600, dtype=torch.complex64)
    a = BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T)
    b = BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T)
    assert torch.equal(a.W, b.W) and torch.equal(a.sum_se, b.sum_se) and torch.equal(a.gamma, b.gamma)
    sub = BT.rzf_batched(H[297:301].contiguous(), wl.alpha(), wl.power(), method=method, T=wl.T)
    assert torch.equal(sub.W, a.W[297:301]) and torch.equal(sub.sum_se, a.sum_se[297:301])


def test_concurrent_streams_use_separate_workspaces():
    """Two batches precoded concurrently on two streams (the per-stream
    workspace cache): results identical to the serial runs."""
    m = X.ChannelModel(S=16, K=64, p=0.4, r=0.7)
    H1 = X.generate_channels(m, seed=31, first=0, B=300, dtype=torch.complex64)
    H2 = X.generate_channels(m, seed=32, first=0, B=300, dtype=torch.complex64)
    ref1 = BT.rzf_batched(H1, 6.4, 10.0, T=4)
    ref2 = BT.rzf_batched(H2, 6.4, 10.0, T=4)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        o1 = BT.rzf_batched(H1, 6.4, 10.0, T=4, check=False, stream=s1)
    with torch.cuda.stream(s2):
        o2 = BT.rzf_batched(H2, 6.4, 10.0, T=4, check=False, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(o1.W, ref1.W) and torch.equal(o2.W, ref2.W)
    assert torch.equal(o1.sum_se, ref1.sum_se) and torch.equal(o2.sum_se, ref2.sum_se)


def test_host_pipeline_reruns_range_rows(monkeypatch):
    """The host-buffer API keeps rzf_batched(check=True)'s contract: a
    realization the fused kernel flags XL_STATUS_RANGE is re-run on the
    general kernels and its W / sum-SE / status scattered back."""
    monkeypatch.setenv("XL_SMALL_K_MMA", "0")  # the tcgen05 kernel (the one that flags RANGE)
    m = X.ChannelModel(S=4, K=16, p=1.0, r=0.5)
    H = X.generate_channels(m, seed=5, first=0, B=5, dtype=torch.complex64)
    H[3, 192:] *= 1e4
    Hh = H.cpu().pin_memory()
    Wh = torch.empty_like(Hh).pin_memory()
    Sh = torch.empty(5, dtype=torch.float64).pin_memory()
    Sth = torch.empty(5, dtype=torch.int32).pin_memory()
    pipe = BT.HostPipeline(m.M, m.K, chunk=2)
    pipe.run(Hh, Wh, Sh, Sth, 1.6, 10.0, "jacpcg", 4)
    assert Sth.tolist() == [0] * 5
    ref = BT.rzf_batched(H, 1.6, 10.0, T=4)
    assert torch.equal(Wh, ref.W.cpu()) and torch.equal(Sh, ref.sum_se.cpu())
    # per-realization xi through the pipeline (sliced per chunk)
    xi = torch.linspace(1.0, 2.0, 5, dtype=torch.float64)
    pipe.run(Hh, Wh, Sh, Sth, xi, 10.0, "jacpcg", 4)
    ref = BT.rzf_batched(H, xi.cuda(), 10.0, T=4)
    assert torch.equal(Wh, ref.W.cpu()) and Sth.tolist() == [0] * 5


def test_out_buffers_and_xi_are_checked():
    """Caller-provided outputs are validated before their pointers reach the
    kernels; per-realization xi must be positive (precoder.py:55-56)."""
    from paper_2305_13925_b200.errors import ConfigurationError
    m = X.ChannelModel(S=4, K=16, p=1.0, r=0.5)
    H = X.generate_channels(m, seed=5, first=0, B=4, dtype=torch.complex64)
    bad = BT.alloc_outputs(H[:3])
    with pytest.raises(ConfigurationError):
        BT.rzf_batched(H, 1.6, 10.0, out=bad)
    wrong = BT.alloc_outputs(H)
    wrong.beta = torch.empty(4, dtype=torch.float32, device=H.device)
    with pytest.raises(ConfigurationError):
        BT.rzf_batched(H, 1.6, 10.0, out=wrong)
    with pytest.raises(ConfigurationError):
        BT.rzf_batched(H, torch.tensor([1.0, 0.0, 1.0, 1.0], device=H.device), 10.0)
    # the range re-run indexes the device copy of a CPU-tensor xi
    H[1, 192:] *= 1e4
    out = BT.rzf_batched(H, torch.tensor([1.6, 1.7, 1.8, 1.9], dtype=torch.float64), 10.0, T=4)
    assert out.status.cpu().tolist() == [0, 0, 0, 0]


@pytest.mark.parametrize("method", ["jacpcg", "cg", "direct"])
def test_rzf_traced_telemetry_vs_oracle(method):
    """xl_rzf_traced: W / SE as xl_rzf plus SolverOutcome's iterations and
    residual_trace (linsolve.py:60-68, _ls_error :89-91) against the oracle."""
    m = X.ChannelModel(S=4, K=32, p=0.5, r=0.5)
    H = X.generate_channels(m, seed=12, first=0, B=3, dtype=torch.complex64)
    alpha, power, T = 3.2, 10.0, 4
    out = BT.rzf_batched(H, alpha, power, method=method, T=T, want_trace=True)
    ref = BT.rzf_batched(H, alpha, power, method=method, T=T)
    if method != "cg":  # unpreconditioned CG: two fp32-level executions differ more (see _check)
        assert relf(out.W.cpu().numpy(), ref.W.cpu().numpy()) < 1e-5
    Hn = H.cpu().numpy().astype(np.complex128)
    its, tr = out.iterations.cpu().numpy(), out.trace.cpu().numpy()
    assert tr.shape == (3, 1 if method == "direct" else T + 1)
    for b in range(3):
        P = O.gram_regularized(Hn[b], alpha)
        I = np.eye(P.shape[0], dtype=complex)
        if method == "direct":
            o = O.direct_solve(P, I)
        elif method == "cg":
            o = O.cg_solve(P, I, T)
        else:
            o = O.jacpcg_solve(P, I, T, variant="textbook")
        assert its[b] == o.iterations
        np.testing.assert_allclose(tr[b], o.residual_trace, rtol=2e-3, atol=1e-10)
    _check(H, out, alpha, power, method, T, "textbook")
