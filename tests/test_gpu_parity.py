"""GPU parity: the CUDA path vs the reference's golden vectors and the CPU oracle.

Tolerances (north_star): W relative Frobenius <= 1e-10 (complex128) and
<= 1e-4 (complex64); sum-SE relative <= 1e-4.  Integer / status outputs and
the CG == Jac-PCG(C=I) identity are bit-exact.
"""

import numpy as np
import pytest
import torch

from oracle import xlmimo_oracle as O

pytestmark = pytest.mark.gpu

import paper_2305_13925_b200 as X  # noqa: E402
from paper_2305_13925_b200 import batched as BT  # noqa: E402
from paper_2305_13925_b200.errors import (ConfigurationError, DegenerateChannelError,  # noqa: E402
                                          NotHpdError, SplittingError)

DEV = "cuda"


def relf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a, dt=torch.complex128):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dt)


# ---------------------------------------------------------------- Gram ------

def test_gram_golden_and_pins(golden):
    g = golden("precoders")
    for tag in ("cfg1", "small", "rand"):
        H = g[tag + "_H"]
        A = BT.gram_batched(dev(H), float(g[tag + "_alpha"])).cpu().numpy()
        ref = g[tag + "_gram"]
        assert relf(A, ref) < 1e-14
        np.testing.assert_array_equal(A, np.conj(np.transpose(A, (0, 2, 1))))  # exact Hermitian
    # test_precoder.py:14-31
    np.testing.assert_array_equal(X.gram_regularized(np.zeros((4, 3)), 0.5).P, 0.5 * np.eye(3))
    np.testing.assert_array_equal(X.gram_regularized(np.eye(2), 1.0).P, 2.0 * np.eye(2))
    with pytest.raises(ConfigurationError):
        X.gram_regularized(np.eye(2), 0.0)


# -------------------------------------------------------------- solvers -----

def _sensitivity(P, S, T, w0, name):
    """Relative change of the ORACLE's answer under a 1e-16 relative Hermitian
    perturbation of P: the round-off floor any implementation inherits.  The
    paper's Algorithm-1 variant diverges on ill-conditioned systems
    and amplifies round-off to ~1e-8 on some golden cases."""
    fns = {"textbook": lambda Q: O.jacpcg_solve(Q, S, T, w0=w0, variant="textbook"),
           "algorithm": lambda Q: O.jacpcg_solve(Q, S, T, w0=w0, variant="algorithm"),
           "cg": lambda Q: O.cg_solve(Q, S, T, w0=w0),
           "eps": lambda Q: O.jacpcg_solve(Q, S, 50, eps=1e-6, w0=w0, variant="textbook")}
    base = fns[name](P).w
    worst = 0.0
    for seed in range(3):
        rng = np.random.default_rng(seed)
        E = rng.standard_normal(P.shape) * 1e-16 * np.abs(P)
        E = (E + E.T) / 2
        worst = max(worst, relf(fns[name](P + E).w, base))
    return worst


def _iterate_sensitivity(P, S, T, w0, name):
    """Per-iterate version of _sensitivity (keep_iterates runs)."""
    fns = {"textbook": lambda Q: O.jacpcg_solve(Q, S, T, w0=w0, variant="textbook", keep_iterates=True),
           "algorithm": lambda Q: O.jacpcg_solve(Q, S, T, w0=w0, variant="algorithm", keep_iterates=True),
           "cg": lambda Q: O.cg_solve(Q, S, T, w0=w0, keep_iterates=True)}
    base = fns[name](P).iterates
    worst = np.zeros(len(base))
    for seed in range(3):
        rng = np.random.default_rng(seed)
        E = rng.standard_normal(P.shape) * 1e-16 * np.abs(P)
        E = (E + E.T) / 2
        its = fns[name](P + E).iterates
        for t in range(min(len(its), len(base))):
            worst[t] = max(worst[t], relf(its[t], base[t]))
    return worst


def test_solver_golden(golden):
    g = golden("solvers")
    for i in range(int(g["n_solver_cases"])):
        pre = f"s{i}_"
        P, S, T = g[pre + "P"], g[pre + "S"], int(g[pre + "T"])
        w0 = g[pre + "w0"] if pre + "w0" in g else None
        sysm = X.HpdSystem(P=P, rhs=S)
        runs = {
            "textbook": lambda: X.jacpcg_solve(sysm, T, w0=w0, keep_iterates=True, variant="textbook"),
            "algorithm": lambda: X.jacpcg_solve(sysm, T, w0=w0, keep_iterates=True, variant="algorithm"),
            "cg": lambda: X.cg_solve(sysm, T, w0=w0, keep_iterates=True),
            "eps": lambda: X.jacpcg_solve(sysm, 50, eps=1e-6, w0=w0, variant="textbook"),
        }
        for name, fn in runs.items():
            if pre + name + "_err" in g:
                with pytest.raises(NotHpdError):
                    fn()
                continue
            o = fn()
            ref_w = g[pre + name + "_w"]
            tol = max(1e-10, 50 * _sensitivity(P, S, T, w0, name))
            assert relf(o.w, ref_w) < tol, (i, name, relf(o.w, ref_w), tol)
            assert o.iterations == int(g[pre + name + "_it"]), (i, name)
            assert o.converged == bool(g[pre + name + "_conv"]), (i, name)
            tr, rtr = o.residual_trace, g[pre + name + "_trace"]
            assert tr.shape == rtr.shape
            # trace values: relative where they are not at round-off level
            np.testing.assert_allclose(tr, rtr, rtol=1e-6, atol=1e-12 * np.nanmax(rtr) + 1e-20)
            if pre + name + "_iterates" in g:
                ri = g[pre + name + "_iterates"]
                assert len(o.iterates) == ri.shape[0]
                sens = _iterate_sensitivity(P, S, T, w0, name)
                for t, (a, b) in enumerate(zip(o.iterates, ri)):
                    assert relf(a, b) < max(tol, 50 * sens[t]), (i, name, t, relf(a, b), sens[t])
        o = X.direct_solve(sysm)
        assert relf(o.w, g[pre + "direct_w"]) < 1e-11
        assert o.iterations == 0 and o.converged


def test_cg_equals_jacpcg_identity_bit_exact():
    """test_linsolve.py:154-164 and acceptance criterion 5(b), on the GPU."""
    rng = np.random.default_rng(9)
    for n in (4, 10, 32):
        A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        Q, _ = np.linalg.qr(A)
        P = (Q * rng.uniform(1, 100, n)) @ Q.conj().T
        P = (P + P.conj().T) / 2
        s = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        sysm = X.HpdSystem(P=P, rhs=s)
        cg = X.cg_solve(sysm, T=6, keep_iterates=True)
        for variant in ("algorithm", "textbook"):
            pcg = X.jacpcg_solve(sysm, T=6, precond_diag=np.ones(n), keep_iterates=True,
                                 variant=variant)
            for a, b in zip(cg.iterates, pcg.iterates):
                np.testing.assert_array_equal(a, b)


def test_solver_known_answers():
    # test_linsolve.py:39-46, 126-134, 166-169
    o = X.direct_solve(X.HpdSystem(P=np.eye(3), rhs=np.array([1.0, 0.0, 0.0])))
    np.testing.assert_allclose(o.w, [1.0, 0.0, 0.0])
    o = X.direct_solve(X.HpdSystem(P=np.diag([2.0, 4.0]), rhs=np.array([2.0, 8.0])))
    np.testing.assert_allclose(o.w, [1.0, 2.0])
    o = X.cg_solve(X.HpdSystem(P=np.eye(4), rhs=np.array([1.0, 2.0, 3.0, 4.0])), T=1)
    np.testing.assert_allclose(o.w, [1.0, 2.0, 3.0, 4.0], atol=1e-14)
    o = X.cg_solve(X.HpdSystem(P=np.eye(3), rhs=np.zeros(3)), T=5)
    np.testing.assert_array_equal(o.w, 0.0)
    o = X.jacpcg_solve(X.HpdSystem(P=np.diag([1.0, 10.0, 100.0]), rhs=np.ones(3)), T=1)
    assert o.residual_trace[-1] < 1e-28
    # multi-RHS == column solves (test_linsolve.py:191-199)
    rng = np.random.default_rng(11)
    A = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    P = A @ A.conj().T + 8 * np.eye(8)
    S = rng.standard_normal((8, 3)) + 1j * rng.standard_normal((8, 3))
    joint = X.jacpcg_solve(X.HpdSystem(P=P, rhs=S), T=5)
    for j in range(3):
        single = X.jacpcg_solve(X.HpdSystem(P=P, rhs=S[:, j]), T=5)
        np.testing.assert_allclose(joint.w[:, j], single.w, rtol=1e-12, atol=1e-14)


def test_solver_errors():
    with pytest.raises(NotHpdError):
        X.direct_solve(X.HpdSystem(P=np.diag([1.0, -1.0]), rhs=np.ones(2)))
    with pytest.raises(NotHpdError):
        X.cg_solve(X.HpdSystem(P=np.diag([1.0, -1.0]), rhs=np.array([0.0, 1.0])), 2)
    with pytest.raises(SplittingError):
        X.jacpcg_solve(X.HpdSystem(P=np.diag([0.0, 1.0]), rhs=np.ones(2)), T=1)
    with pytest.raises(ConfigurationError):
        X.jacpcg_solve(X.HpdSystem(P=np.eye(2), rhs=np.ones(2)), T=1, variant="fast")
    with pytest.raises(ConfigurationError):
        X.cg_solve(X.HpdSystem(P=np.eye(2), rhs=np.ones(2)), T=0)
    # batched: a bad realization is flagged per realization, others untouched
    A = torch.eye(3, dtype=torch.complex128, device=DEV).repeat(3, 1, 1)
    A[1, 2, 2] = -1.0
    res = BT.solve_batched(A, "cg", T=3, check=False)
    assert res.status.cpu().tolist() == [0, 1, 0]
    res = BT.solve_batched(A, "direct", check=False)
    assert res.status.cpu().tolist() == [0, 4, 0]


# ----------------------------------------------------------- precoders ------

@pytest.mark.parametrize("tag", ["cfg1", "small", "rand"])
def test_precoder_golden_c128(golden, tag):
    g = golden("precoders")
    Hb = g[tag + "_H"]
    alpha, power, sigma2 = float(g[tag + "_alpha"]), float(g[tag + "_power"]), float(g[tag + "_sigma2"])
    H = dev(Hb)
    for key in [k for k in g.files if k.startswith(tag + "_") and k.endswith("_G")]:
        meth_T = key[len(tag) + 1:-2]
        meth, T = meth_T.rsplit("_T", 1)
        method = meth.split("_")[0]
        variant = meth.split("_")[1] if "_" in meth else "textbook"
        out = BT.rzf_batched(H, alpha, power, method=method, T=int(T), variant=variant,
                             sigma2=sigma2, want_F=True)
        W = out.W.cpu().numpy()
        for b in range(Hb.shape[0]):
            assert relf(W[b], g[key][b]) <= 1e-10, (key, b, relf(W[b], g[key][b]))
        np.testing.assert_allclose(out.beta.cpu().numpy(), g[key[:-2] + "_beta"], rtol=1e-10)
        # interference = row total - signal (metrics.py:54) cancels when one user
        # dominates its row, so gamma inherits ~1e-8 relative round-off.
        np.testing.assert_allclose(out.gamma.cpu().numpy(), g[key[:-2] + "_gamma"], rtol=1e-7)
        # SE inherits gamma's cancellation (see above): 1e-8 relative in complex128
        np.testing.assert_allclose(out.sum_se.cpu().numpy(), g[key[:-2] + "_sumse"], rtol=1e-8)
        # G = beta F (precoder.py:70)
        np.testing.assert_allclose(W, out.F.cpu().numpy() * out.beta.cpu().numpy()[:, None, None],
                                   rtol=1e-14, atol=0)


def test_precoder_mirror_pins():
    """test_precoder.py:38-103 through the reference-named mirror."""
    power = 3.0
    blk = X.rzf_direct(np.eye(2), 1.0, power)
    np.testing.assert_allclose(blk.F, 0.5 * np.eye(2), atol=1e-14)
    assert blk.beta == pytest.approx(np.sqrt(power / 0.5))
    rng = np.random.default_rng(2)
    H = rng.standard_normal((12, 6)) + 1j * rng.standard_normal((12, 6))
    blk = X.rzf_direct(H, 0.3, 2.5)
    assert float(np.vdot(blk.G, blk.G).real) == pytest.approx(2.5, rel=1e-10)
    H = rng.standard_normal((10, 4)) + 1j * rng.standard_normal((10, 4))
    blk = X.rzf_direct(H, 1e6, 1.0)   # matched-filter limit
    assert np.linalg.norm(blk.G / np.linalg.norm(blk.G) - H / np.linalg.norm(H)) < 1e-3
    with pytest.raises(DegenerateChannelError):
        X.rzf_direct(np.zeros((4, 2)), 0.5, 1.0)
    H = np.random.default_rng(4).standard_normal((12, 6)) + 1j * np.random.default_rng(5).standard_normal((12, 6))
    exact = X.rzf_direct(H, 0.2, 1.0)
    approx = X.rzf_iterative(H, 0.2, 1.0, solver="cg", T=6)
    assert np.linalg.norm(approx.G - exact.G) / np.linalg.norm(exact.G) < 1e-6
    for solver in ("cg", "jacpcg"):
        blk = X.rzf_iterative(H, 0.2, 4.0, solver=solver, T=3, pcg_variant="textbook")
        assert float(np.vdot(blk.G, blk.G).real) == pytest.approx(4.0, rel=1e-10)
    errs = [np.linalg.norm(X.rzf_iterative(H, 0.2, 1.0, solver="cg", T=T).G - exact.G)
            for T in range(1, 7)]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(errs, errs[1:]))
    with pytest.raises(ConfigurationError):
        X.rzf_iterative(H, 0.2, 1.0, solver="cg", T=0)
    with pytest.raises(ConfigurationError):
        X.rzf_iterative(H, 0.2, 1.0, solver="sor", T=2)
    # eps early stop path matches the oracle
    ref = O.rzf_iterative(H, 0.2, 1.0, "jacpcg", 50, eps=1e-8, pcg_variant="textbook")
    blk = X.rzf_iterative(H, 0.2, 1.0, solver="jacpcg", T=50, eps=1e-8, pcg_variant="textbook")
    assert relf(blk.G, ref[0]) < 1e-10


def test_sinr_mirror_pins():
    rng = np.random.default_rng(0)
    H = rng.standard_normal((9, 4)) + 1j * rng.standard_normal((9, 4))
    G, _, _ = O.rzf_direct(H, 0.5, 1.0)
    rep = X.sinr_eq9(H, G, 1e-9)
    g_ref, se_ref, s_ref = O.sinr_single_block(H, G, 1e-9)
    np.testing.assert_allclose(rep.gamma, g_ref, rtol=1e-12)
    assert rep.sum_se == pytest.approx(rep.se_per_user.sum())
    np.testing.assert_allclose(X.coupling_matrix(H, G), H.conj().T @ G, atol=1e-12)
    zero = X.sinr_eq9(H, np.zeros_like(G), 1e-8)
    np.testing.assert_array_equal(zero.gamma, 0.0)
    assert zero.sum_se == 0.0
    with pytest.raises(ConfigurationError):
        X.sinr_eq9(H, G, 0.0)
    assert X.sum_se([5.0]) == (5.0, 0.0)
    m, s = X.sum_se(torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64, device=DEV))
    assert m == pytest.approx(2.0) and s == pytest.approx(1.0 / np.sqrt(3.0))


# ------------------------------------------------------- complex64 path -----

@pytest.mark.parametrize("cfg,B", [("cfg2", 16), ("cfg3", 8), ("cfg4", 2)])
@pytest.mark.parametrize("method", ["jacpcg", "cg", "direct"])
def test_c64_vs_oracle(cfg, B, method):
    wl = X.CONFIGS[cfg]
    H = X.generate_channels(wl.model, seed=0, first=1000, B=B, dtype=torch.complex64)
    out = BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T, sigma2=1.0)
    Hn = H.cpu().numpy().astype(np.complex128)   # input quantisation not charged to the kernel
    W = out.W.cpu().numpy()
    S = out.sum_se.cpu().numpy()
    for b in range(B):
        Gr, beta, gam, s = O.precoder_and_se(Hn[b], wl.alpha(), wl.power(), 1.0, method, wl.T,
                                             "textbook")
        assert relf(W[b], Gr) <= 1e-4, (cfg, method, b, relf(W[b], Gr))
        assert abs(S[b] - s) / abs(s) <= 1e-4, (cfg, method, b, S[b], s)


@pytest.mark.parametrize("cfg,B,tol", [("cfg5", 2, 1e-4), ("cfg5_c128", 1, 1e-10), ("cfg4", 3, 1e-4)])
def test_large_k_tensor_core_general_path(cfg, B, tol):
    """K >= 96: the general path's Gram and W run on the tensor cores
    (3xTF32 for complex64, ZGEMM for complex128; gemm_tc.cu), in sub-batches."""
    wl = X.CONFIGS[cfg]
    H = X.generate_channels(wl.model, seed=2, first=77, B=B, dtype=wl.dtype)
    Hn = H.cpu().numpy().astype(np.complex128)
    for method in ("jacpcg", "direct"):
        out = BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T, want_F=True)
        W, F, S = out.W.cpu().numpy(), out.F.cpu().numpy(), out.sum_se.cpu().numpy()
        beta, gam = out.beta.cpu().numpy(), out.gamma.cpu().numpy()
        for b in range(B):
            Gr, br, gr, s = O.precoder_and_se(Hn[b], wl.alpha(), wl.power(), 1.0, method, wl.T, "textbook")
            assert relf(W[b], Gr) <= tol, (cfg, method, b, relf(W[b], Gr))
            assert relf(F[b], Gr / br) <= tol, (cfg, method, b)
            assert abs(beta[b] - br) <= tol * br
            assert abs(S[b] - s) <= max(tol, 1e-8) * abs(s), (cfg, method, b, S[b], s)
            np.testing.assert_allclose(gam[b], gr, rtol=max(10 * tol, 1e-8))


@pytest.mark.parametrize("M,K", [(1000, 96), (640, 320), (130, 128)])
def test_large_k_odd_shapes(M, K):
    """Tensor-core general path at shapes off the BASELINE grid: K = 96 (n2 not a
    multiple of 128), K = 320 (tensor-core Gram / W with the SIMT Jac-PCG), M not a
    multiple of 64, per-realization xi."""
    rng = np.random.default_rng(M + K)
    Hn = (rng.standard_normal((2, M, K)) + 1j * rng.standard_normal((2, M, K))) / np.sqrt(2)
    H = torch.from_numpy(Hn.astype(np.complex64)).to(DEV)
    xi = torch.tensor([K / 10.0, K / 3.0], dtype=torch.float64, device=DEV)
    out = BT.rzf_batched(H, xi, 10.0, method="jacpcg", T=4)
    Hq = H.cpu().numpy().astype(np.complex128)
    for b in range(2):
        Gr, br, gr, s = O.precoder_and_se(Hq[b], float(xi[b]), 10.0, 1.0, "jacpcg", 4, "textbook")
        assert relf(out.W[b].cpu().numpy(), Gr) <= 1e-4, (M, K, b)
        assert abs(out.sum_se[b].item() - s) <= 1e-4 * abs(s)


def test_large_k_pcg_variants_vs_oracle():
    """The tensor-core Jac-PCG / CG of the large-K general path (gemm_tc.cu
    tc_pcg) against the complex128 oracle for all three recurrences on the
    same regularized Gram matrices; Algorithm 1 amplifies round-off (SURVEY
    F2), so its bound is looser."""
    wl = X.CONFIGS["cfg4"]
    H = X.generate_channels(wl.model, seed=5, first=3, B=2, dtype=torch.complex64)
    Hn = H.cpu().numpy().astype(np.complex128)
    for method, variant, tol in (("jacpcg", "textbook", 1e-4), ("cg", "textbook", 1e-3),
                                 ("jacpcg", "algorithm", 1e-2)):
        out = BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T, variant=variant,
                             want_X=True)
        Xg = out.X.cpu().numpy()
        for b in range(2):
            P = O.gram_regularized(Hn[b], wl.alpha())
            K = P.shape[0]
            o = (O.cg_solve(P, np.eye(K), wl.T) if method == "cg"
                 else O.jacpcg_solve(P, np.eye(K), wl.T, variant=variant))
            assert relf(Xg[b], o.w) <= tol, (method, variant, b, relf(Xg[b], o.w))
        assert (out.status == 0).all()


def test_large_k_pcg_c128_variants_vs_oracle():
    """complex128 large-K rzf path (ZGEMM Gram / W, ZGEMM-based Jac-PCG / CG and
    GX): all three recurrences at the c128 tolerance."""
    rng = np.random.default_rng(17)
    M, K, T = 512, 128, 5
    Hn = (rng.standard_normal((2, M, K)) + 1j * rng.standard_normal((2, M, K))) / np.sqrt(2)
    H = torch.from_numpy(Hn).to(DEV)
    xi, power = K / 10.0, 10.0
    for method, variant in (("jacpcg", "textbook"), ("cg", "textbook"), ("jacpcg", "algorithm")):
        out = BT.rzf_batched(H, xi, power, method=method, T=T, variant=variant, want_X=True)
        for b in range(2):
            Gr, br, gr, s = O.precoder_and_se(Hn[b], xi, power, 1.0, method, T, variant)
            tol = max(1e-10, 100 * _sensitivity(O.gram_regularized(Hn[b], xi), np.eye(K), T, None,
                                                "cg" if method == "cg" else variant))
            assert relf(out.W[b].cpu().numpy(), Gr) <= tol, (method, variant, b, relf(out.W[b].cpu().numpy(), Gr))
            assert abs(out.sum_se[b].item() - s) <= max(1e-8, tol) * abs(s)
        assert (out.status == 0).all()


def test_c128_cfg1_full_batch():
    """configs[0]: 100 realizations, complex128, Jac-PCG T=4 and direct at 1e-10."""
    wl = X.CONFIGS["cfg1"]
    H = X.generate_channels(wl.model, seed=0, first=0, B=wl.B, dtype=torch.complex128)
    Hn = H.cpu().numpy()
    for method in ("jacpcg", "direct"):
        out = BT.rzf_batched(H, wl.alpha(), wl.power(), method=method, T=wl.T)
        W = out.W.cpu().numpy()
        S = out.sum_se.cpu().numpy()
        for b in range(wl.B):
            Gr, beta, gam, s = O.precoder_and_se(Hn[b], wl.alpha(), wl.power(), 1.0, method,
                                                 wl.T, "textbook")
            assert relf(W[b], Gr) <= 1e-10
            assert abs(S[b] - s) <= 1e-10 * abs(s)


def test_power_identity_and_properties_full_size():
    """Size-independent properties at a BASELINE size (cfg3 shape, 512 realizations)."""
    wl = X.CONFIGS["cfg3"]
    H = X.generate_channels(wl.model, seed=1, first=0, B=512, dtype=torch.complex64)
    out = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T, want_F=True)
    tr = (out.W.abs() ** 2).sum(dim=(1, 2)).double()
    assert torch.allclose(tr, torch.full_like(tr, wl.power()), rtol=1e-5)
    assert (out.gamma >= 0).all() and torch.isfinite(out.gamma).all()
    se = torch.log2(1 + out.gamma).sum(dim=1)
    assert torch.allclose(se, out.sum_se, rtol=1e-12)
    assert (out.status == 0).all()
    # determinism: identical bits on a second run
    out2 = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T)
    assert torch.equal(out.W, out2.W) and torch.equal(out.sum_se, out2.sum_se)
    # batch independence: a sub-batch reproduces the same bits
    sub = BT.rzf_batched(H[100:117].contiguous(), wl.alpha(), wl.power(), T=wl.T)
    assert torch.equal(sub.W, out.W[100:117])


def test_degenerate_realization_flagged():
    H = torch.randn(3, 64, 8, dtype=torch.complex64, device=DEV)
    H[1] = 0
    out = BT.rzf_batched(H, 0.5, 1.0, T=3, check=False)
    assert out.status.cpu().tolist() == [0, 3, 0]
    with pytest.raises(DegenerateChannelError):
        BT.rzf_batched(H, 0.5, 1.0, T=3)


# ------------------------------------------------------------- channel ------

@pytest.mark.parametrize("dt,tol", [(torch.complex128, 1e-12), (torch.complex64, 2e-6)])
def test_channel_generator_vs_oracle(dt, tol):
    # cfg4's shape (64 x 128, p = 0.3) and > 64 visible users per subarray (two user chunks
    # on the tensor-core generator, the second one partial)
    for (S, K, p, r, B) in ((4, 16, 0.5, 0.5, 6), (16, 64, 0.4, 0.7, 6), (3, 5, 0.3, 0.9, 6),
                            (64, 128, 0.3, 0.5, 2), (4, 100, 0.95, 0.9, 3)):
        m = X.ChannelModel(S=S, K=K, p=p, r=r)
        H = X.generate_channels(m, seed=123, first=77, B=B, dtype=dt).cpu().numpy()
        ref = O.generate_channels(123, 77, B, S, K, p, r)
        # exact zeros on invisible subarrays
        np.testing.assert_array_equal(H == 0, ref == 0)
        assert relf(H, ref) < tol


def test_channel_sharding_property():
    m = X.ChannelModel(S=16, K=64, p=0.4, r=0.7)
    full = X.generate_channels(m, seed=5, first=0, B=64)
    a = X.generate_channels(m, seed=5, first=0, B=32)
    b = X.generate_channels(m, seed=5, first=32, B=32)
    assert torch.equal(torch.cat([a, b]), full)


def test_se_partials_vs_oracle():
    x = torch.rand(10000, dtype=torch.float64, device=DEV) * 50
    parts = BT.se_partials(x, 2048).cpu().numpy()
    assert parts.shape == (5, 3) and parts[:, 2].sum() == 10000
    mean, sem = BT.combine_se_partials(parts)
    rm, rs = O.sum_se(x.cpu().numpy())
    assert mean == pytest.approx(rm, rel=1e-13) and sem == pytest.approx(rs, rel=1e-9)
    # the device combine (xl_se_combine, one launch) sums the partials in the
    # same chunk order as the host combine
    from paper_2305_13925_b200.distributed import combine_partials_device, ergodic_se
    dm, ds = combine_partials_device(BT.se_partials(x, 2048))
    assert float(dm) == mean and float(ds) == pytest.approx(sem, rel=1e-14)
    em, es = ergodic_se(x[:1], chunk=2048, group=False)  # one realization: SEM 0
    assert float(em) == float(x[0]) and float(es) == 0.0


@pytest.mark.parametrize("cfg,B", [("cfg1", 100), ("cfg2", 300), ("cfg3", 64), ("cfg4", 4), ("cfg5", 1100)])
def test_graphed_rzf_matches_direct_calls(cfg, B):
    """CUDA-graph replay of the whole precoder chain (fused kernel, SIMT general
    path, the K = 128 tcgen05 chain with its 2-CTA clusters and DSMEM bulk
    copies, the small-K kernel with its TMEM allocation and W tensor map, the
    K = 256 chain's chunks forked onto a second stream and joined back)
    gives the same bits as the direct call, on two different inputs."""
    wl = X.CONFIGS[cfg]
    g = BT.GraphedRzf(B, wl.M, wl.K, wl.dtype, wl.alpha(), wl.power(), T=wl.T)
    for seed in (0, 1):
        H = X.generate_channels(wl.model, seed=seed, first=0, B=B, dtype=wl.dtype)
        ref = BT.rzf_batched(H, wl.alpha(), wl.power(), T=wl.T)
        out = g.run(H)
        assert torch.equal(out.W, ref.W) and torch.equal(out.sum_se, ref.sum_se)
        assert torch.equal(out.beta, ref.beta)
