"""GPU parity of the fused 2-CTA-cluster Jac-PCG (cluster_pcg.cu, K = 128
complex64) that the large-K rzf path uses in place of the split-GEMM solver.

Checks: W / beta / SE against the complex128 oracle (north_star tolerances,
W relative Frobenius <= 1e-4), agreement with the split-GEMM solver it
replaces (XL_LARGE_K_SOLVER=gemm selects that one per call), bit-identical
repeat calls (the pair's scalars are summed in a fixed order), many clusters
per launch, and per-realization xi.
"""

import os

import numpy as np
import pytest
import torch

from oracle import xlmimo_oracle as O

pytestmark = pytest.mark.gpu

import paper_2305_13925_b200 as X  # noqa: E402
from paper_2305_13925_b200 import batched as BT  # noqa: E402

DEV = "cuda"


def relf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _run(H, xi, power, method="jacpcg", T=5, variant="textbook", solver=None, **kw):
    old = os.environ.get("XL_LARGE_K_SOLVER")
    try:
        if solver:
            os.environ["XL_LARGE_K_SOLVER"] = solver
        else:
            os.environ.pop("XL_LARGE_K_SOLVER", None)
        out = BT.rzf_batched(H, xi, power, method=method, T=T, variant=variant, **kw)
        torch.cuda.synchronize()
        return out
    finally:
        if old is None:
            os.environ.pop("XL_LARGE_K_SOLVER", None)
        else:
            os.environ["XL_LARGE_K_SOLVER"] = old


@pytest.mark.parametrize("method,variant,tol", [("jacpcg", "textbook", 1e-4), ("cg", "textbook", 1e-3),
                                                ("jacpcg", "algorithm", 1e-2)])
def test_cluster_pcg_vs_oracle_cfg4_channel(method, variant, tol):
    wl = X.CONFIGS["cfg4"]
    H = X.generate_channels(wl.model, seed=11, first=5, B=3, dtype=torch.complex64)
    Hn = H.cpu().numpy().astype(np.complex128)
    out = _run(H, wl.alpha(), wl.power(), method=method, T=wl.T, variant=variant, want_X=True)
    W, S, beta = out.W.cpu().numpy(), out.sum_se.cpu().numpy(), out.beta.cpu().numpy()
    assert (out.status.cpu().numpy() == 0).all()
    for b in range(3):
        Gr, br, gr, s = O.precoder_and_se(Hn[b], wl.alpha(), wl.power(), 1.0, method, wl.T, variant)
        assert relf(W[b], Gr) <= tol, (method, variant, b, relf(W[b], Gr))
        assert abs(beta[b] - br) <= tol * br
        assert abs(S[b] - s) <= max(tol, 1e-4) * abs(s), (method, variant, b, S[b], s)


def test_cluster_pcg_matches_split_gemm_solver():
    """Same Gram, two solvers: the on-chip cluster solver and the split-GEMM
    tc_pcg + tc_gx chain agree to the 3xFP16 / 3xTF32 rounding level."""
    rng = np.random.default_rng(7)
    B, M, K = 40, 384, 128
    Hn = (rng.standard_normal((B, M, K)) + 1j * rng.standard_normal((B, M, K))) / np.sqrt(2)
    H = torch.from_numpy(Hn.astype(np.complex64)).to(DEV)
    xi = torch.from_numpy(rng.uniform(K / 30, K / 3, size=B)).to(DEV)
    a = _run(H, xi, 10.0, T=5, want_X=True)
    g = _run(H, xi, 10.0, T=5, want_X=True, solver="gemm")
    for b in range(B):
        assert relf(a.X[b].cpu().numpy(), g.X[b].cpu().numpy()) <= 2e-5, b
        assert relf(a.W[b].cpu().numpy(), g.W[b].cpu().numpy()) <= 2e-5, b
    np.testing.assert_allclose(a.beta.cpu().numpy(), g.beta.cpu().numpy(), rtol=2e-5)
    np.testing.assert_allclose(a.sum_se.cpu().numpy(), g.sum_se.cpu().numpy(), rtol=2e-5)
    np.testing.assert_allclose(a.gamma.cpu().numpy(), g.gamma.cpu().numpy(), rtol=1e-4)
    # spot-check against the oracle with the per-realization xi
    Hq = H.cpu().numpy().astype(np.complex128)
    for b in (0, B - 1):
        Gr, br, gr, s = O.precoder_and_se(Hq[b], float(xi[b]), 10.0, 1.0, "jacpcg", 5, "textbook")
        assert relf(a.W[b].cpu().numpy(), Gr) <= 1e-4
        assert abs(a.sum_se[b].item() - s) <= 1e-4 * abs(s)


def test_cluster_pcg_deterministic_and_many_clusters():
    """Hundreds of clusters (several waves) and bit-identical repeat calls."""
    wl = X.CONFIGS["cfg4"]
    rng = np.random.default_rng(3)
    B, M, K = 300, 256, 128
    Hn = (rng.standard_normal((B, M, K)) + 1j * rng.standard_normal((B, M, K))) / np.sqrt(2)
    H = torch.from_numpy(Hn.astype(np.complex64)).to(DEV)
    o1 = _run(H, wl.alpha(), wl.power(), T=5, want_X=True)
    o2 = _run(H, wl.alpha(), wl.power(), T=5, want_X=True)
    assert torch.equal(o1.X, o2.X) and torch.equal(o1.W, o2.W)
    assert torch.equal(o1.sum_se, o2.sum_se) and torch.equal(o1.beta, o2.beta)
    Hq = H.cpu().numpy().astype(np.complex128)
    for b in (0, 149, 299):
        Gr, br, gr, s = O.precoder_and_se(Hq[b], wl.alpha(), wl.power(), 1.0, "jacpcg", 5, "textbook")
        assert relf(o1.W[b].cpu().numpy(), Gr) <= 1e-4, b


def _run_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    try:
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        out = fn()
        torch.cuda.synchronize()
        return out
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("method", ["jacpcg", "direct"])
def test_streaming_gram_w_match_library_gemms(method):
    """stream_tc.cu (tcgen05 Gram / W with the in-smem 3xFP16 split) against the
    split-operand library GEMMs it replaces (XL_LARGE_K_GEMM=library) and the
    complex128 oracle; F = W / beta, a wide per-user gain spread (the per-row X
    scales), a realization whose later antennas overflow the first chunk's
    fp16 scale (flag + fixup launch) and one with leading zero chunks."""
    rng = np.random.default_rng(21)
    B, M, K = 6, 640, 128
    Hn = (rng.standard_normal((B, M, K)) + 1j * rng.standard_normal((B, M, K))) / np.sqrt(2)
    Hn *= 10.0 ** rng.uniform(-2, 1, size=(B, 1, K))  # 60 dB of user gain spread
    Hn[1] *= 1e-6                                      # a tiny realization (scale 2^e far from 1)
    Hn[2, 256:] *= 300.0                               # later chunks overflow the first chunk's scale: fixup
    Hn[3, :128] = 0.0                                  # leading zero chunks: scale from the first non-zero one
    H = torch.from_numpy(Hn.astype(np.complex64)).to(DEV)
    xi = torch.from_numpy(rng.uniform(0.05, 2.0, size=B) * np.abs(Hn).mean(axis=(1, 2)) ** 2 * M).to(DEV)
    f = lambda: BT.rzf_batched(H, xi, 10.0, method=method, T=6, want_F=True, want_X=True)
    s = _run_env({"XL_LARGE_K_GEMM": None}, f)
    lib = _run_env({"XL_LARGE_K_GEMM": "library"}, f)
    Hq = H.cpu().numpy().astype(np.complex128)
    for b in range(B):
        Gr, br, gr, se = O.precoder_and_se(Hq[b], float(xi[b]), 10.0, 1.0, method, 6, "textbook")
        Ws, Wl = s.W[b].cpu().numpy(), lib.W[b].cpu().numpy()
        assert relf(Ws, Gr) <= 1e-4, (b, relf(Ws, Gr))
        assert relf(Ws, Wl) <= 2e-5, (b, relf(Ws, Wl))
        assert relf(s.F[b].cpu().numpy(), Gr / br) <= 1e-4
        assert abs(s.beta[b].item() - br) <= 1e-4 * br
        assert abs(s.sum_se[b].item() - se) <= 1e-4 * abs(se)


@pytest.mark.parametrize("B,M,T", [(1, 64, 1), (3, 64, 2), (4100, 64, 3)])
def test_k128_edge_shapes(B, M, T):
    """One 64-antenna chunk, T = 1, a single realization, and a batch past the
    streaming Gram's 4096-realization sub-batch (U workspace reuse)."""
    K = 128
    g = torch.Generator(device=DEV).manual_seed(B + M + T)
    H = torch.complex(torch.randn(B, M, K, device=DEV, generator=g),
                      torch.randn(B, M, K, device=DEV, generator=g)) * 0.7
    H = H.to(torch.complex64)
    xi = K / 10.0
    out = _run(H, xi, 10.0, T=T)
    assert (out.status.cpu().numpy() == 0).all()
    Hq = H.cpu().numpy().astype(np.complex128)
    for b in sorted({0, B // 2, B - 1}):
        Gr, br, gr, s = O.precoder_and_se(Hq[b], xi, 10.0, 1.0, "jacpcg", T, "textbook")
        assert relf(out.W[b].cpu().numpy(), Gr) <= 1e-4, (B, M, T, b)
        assert abs(out.sum_se[b].item() - s) <= 1e-4 * abs(s)


def test_k128_pair_w_kernel_matches_single_cta():
    """The K = 128 W product as a cta_group::2 pair (default) against the
    single-CTA w_kernel (XL_STREAM_W2=0): W / F within fp32 rounding, sum-SE too."""
    import os
    wl = X.CONFIGS["cfg4"]
    H = X.generate_channels(wl.model, seed=3, first=9, B=6, dtype=torch.complex64)
    run = lambda: BT.rzf_batched(H, wl.alpha(), wl.power(), T=5, want_F=True)  # noqa: E731
    ref = run()
    torch.cuda.synchronize()
    os.environ["XL_STREAM_W2"] = "0"
    try:
        alt = run()
        torch.cuda.synchronize()
    finally:
        os.environ.pop("XL_STREAM_W2", None)
    for b in range(H.shape[0]):
        w0, w1 = ref.W[b].cpu().numpy(), alt.W[b].cpu().numpy()
        assert np.linalg.norm(w0 - w1) <= 2e-5 * np.linalg.norm(w1)
        f0, f1 = ref.F[b].cpu().numpy(), alt.F[b].cpu().numpy()
        assert np.linalg.norm(f0 - f1) <= 2e-5 * np.linalg.norm(f1)
    assert torch.equal(ref.sum_se, alt.sum_se)  # SINR comes from the solver, not from W
