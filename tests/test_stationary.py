"""Stationary splittings JOR / Gauss-Seidel.

CPU: the oracle restatement (oracle/xlmimo_oracle.py jor_solve / gs_solve) vs
the golden vectors written from the live reference (linsolve.py:128-176).
GPU: xl_solve_stationary through the reference-shaped API (complex128) vs the
same vectors, the batched complex64 path vs the oracle, and the error paths.
"""

import numpy as np
import pytest

from oracle import xlmimo_oracle as O

RUNS = {
    "jor05": lambda f, P, S, T, w0: f["jor"](P, S, T, omega=0.5, w0=w0, keep_iterates=True),
    "jor10": lambda f, P, S, T, w0: f["jor"](P, S, T, omega=1.0, w0=w0, keep_iterates=True),
    "gs": lambda f, P, S, T, w0: f["gs"](P, S, T, w0=w0, keep_iterates=True),
    "gseps": lambda f, P, S, T, w0: f["gs"](P, S, 40, w0=w0, eps=1e-5),
}
ORACLE = {"jor": O.jor_solve, "gs": O.gs_solve}


def relf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def _cases(g):
    for i in range(int(g["n_cases"])):
        pre = f"s{i}_"
        yield pre, g[pre + "P"], g[pre + "S"], int(g[pre + "T"]), (g[pre + "w0"] if pre + "w0" in g else None)


def test_oracle_stationary_golden(golden):
    g = golden("stationary")
    assert int(g["n_cases"]) == 24
    for pre, P, S, T, w0 in _cases(g):
        for name, run in RUNS.items():
            o = run(ORACLE, P, S, T, w0)
            w, tr = g[pre + name + "_w"], g[pre + name + "_trace"]
            if name.startswith("jor"):  # the same numpy expression as the reference: bit-exact
                np.testing.assert_array_equal(o.w, w)
                np.testing.assert_array_equal(o.residual_trace, tr)
            else:  # explicit forward substitution vs scipy's trsm: round-off only
                assert relf(o.w, w) < 1e-12, (pre, name, relf(o.w, w))
                np.testing.assert_allclose(o.residual_trace, tr, rtol=1e-8, atol=1e-13)
            assert o.iterations == int(g[pre + name + "_it"])
            assert o.converged == bool(g[pre + name + "_conv"])
            if pre + name + "_iterates" in g:
                ri = g[pre + name + "_iterates"]
                assert len(o.iterates) == ri.shape[0]
                for a, b in zip(o.iterates, ri):
                    assert relf(a, b) < 1e-12


def test_oracle_stationary_errors(golden):
    g = golden("stationary")
    cases = {
        "gs_zero_diag": lambda: O.gs_solve(np.diag([0.0, 1.0]), np.ones(2), 1),
        "jor_zero_diag": lambda: O.jor_solve(np.diag([1.0, 0.0]), np.ones(2), 1),
        "jor_omega": lambda: O.jor_solve(np.eye(2), np.ones(2), 1, omega=0.0),
        "gs_T0": lambda: O.gs_solve(np.eye(2), np.ones(2), 0),
    }
    for name, fn in cases.items():
        with pytest.raises(O.OracleError) as ei:
            fn()
        assert ei.value.kind == str(g["err_" + name])


# ------------------------------------------------------------------ GPU -----

def _api():
    import paper_2305_13925_b200 as X

    def jor(P, S, T, omega=0.5, w0=None, eps=None, keep_iterates=False):
        return X.jor_solve(X.HpdSystem(P=P, rhs=S), T, omega=omega, w0=w0, eps=eps,
                           keep_iterates=keep_iterates)

    def gs(P, S, T, w0=None, eps=None, keep_iterates=False):
        return X.gs_solve(X.HpdSystem(P=P, rhs=S), T, w0=w0, eps=eps, keep_iterates=keep_iterates)
    return {"jor": jor, "gs": gs}


@pytest.mark.gpu
def test_gpu_stationary_golden_c128(golden):
    g = golden("stationary")
    api = _api()
    for pre, P, S, T, w0 in _cases(g):
        for name, run in RUNS.items():
            o = run(api, P, S, T, w0)
            w = g[pre + name + "_w"]
            assert relf(o.w, w) < 1e-10, (pre, name, relf(o.w, w))
            assert o.iterations == int(g[pre + name + "_it"]), (pre, name)
            assert o.converged == bool(g[pre + name + "_conv"]), (pre, name)
            tr = g[pre + name + "_trace"]
            assert o.residual_trace.shape == tr.shape
            np.testing.assert_allclose(o.residual_trace, tr, rtol=1e-6, atol=1e-12 * tr.max() + 1e-20)
            if pre + name + "_iterates" in g:
                ri = g[pre + name + "_iterates"]
                assert len(o.iterates) == ri.shape[0]
                for a, b in zip(o.iterates, ri):
                    assert relf(a, b) < 1e-10


@pytest.mark.gpu
def test_gpu_stationary_errors():
    import paper_2305_13925_b200 as X
    from paper_2305_13925_b200.errors import ConfigurationError, SplittingError
    with pytest.raises(SplittingError):
        X.gs_solve(X.HpdSystem(P=np.diag([0.0, 1.0]), rhs=np.ones(2)), 1)
    with pytest.raises(SplittingError):
        X.jor_solve(X.HpdSystem(P=np.diag([1.0, 0.0]), rhs=np.ones(2)), 1)
    with pytest.raises(ConfigurationError):
        X.jor_solve(X.HpdSystem(P=np.eye(2), rhs=np.ones(2)), 1, omega=0.0)
    with pytest.raises(ConfigurationError):
        X.gs_solve(X.HpdSystem(P=np.eye(2), rhs=np.ones(2)), 0)
    # the device kernel's own zero-diagonal check (status path, no host pre-check)
    import torch
    from paper_2305_13925_b200 import batched as BT
    A = torch.eye(3, dtype=torch.complex128, device="cuda").repeat(2, 1, 1)
    A[1, 2, 2] = 0
    r = BT.solve_batched(A, "gs", T=2, check=False)
    assert r.status.cpu().tolist() == [0, 2]
    with pytest.raises(SplittingError):
        BT.solve_batched(A, "jor", T=2)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["jor", "gs"])
def test_gpu_stationary_batched_c64_vs_oracle(method):
    """Batched complex64 on regularized Gram matrices of BASELINE-model
    channels (cfg2 shape, M = 256, K = 32) against the complex128 oracle."""
    import torch
    import paper_2305_13925_b200 as X
    from paper_2305_13925_b200 import batched as BT
    wl = X.CONFIGS["cfg2"]
    H = X.generate_channels(wl.model, seed=1, first=0, B=16, dtype=torch.complex64)
    A = BT.gram_batched(H, wl.alpha())
    r = BT.solve_batched(A, method, T=5, trace=True, omega=0.7)
    A64 = A.to(torch.complex128).cpu().numpy()
    for b in range(16):
        K = A64.shape[1]
        o = (O.jor_solve(A64[b], np.eye(K), 5, omega=0.7) if method == "jor"
             else O.gs_solve(A64[b], np.eye(K), 5))
        assert relf(r.X[b].cpu().numpy(), o.w) < 1e-5, (b, relf(r.X[b].cpu().numpy(), o.w))
        np.testing.assert_allclose(r.trace[b].cpu().numpy(), o.residual_trace, rtol=1e-3, atol=1e-7)


@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["jor", "gs"])
def test_gpu_rzf_iterative_stationary(solver):
    """rzf_iterative(solver=jor|gs) (precoder.py:81-91 via solve_iterative)
    against the oracle's Gram + solver + H X + power scaling."""
    import paper_2305_13925_b200 as X
    g_rng = np.random.default_rng(4)
    H = g_rng.standard_normal((48, 12)) + 1j * g_rng.standard_normal((48, 12))
    xi, power = 1.2, 10.0
    blk = X.rzf_iterative(H, xi, power, solver=solver, T=4, omega=0.6)
    P = O.gram_regularized(H, xi)
    o = (O.jor_solve(P, np.eye(12), 4, omega=0.6) if solver == "jor" else O.gs_solve(P, np.eye(12), 4))
    F = H @ o.w
    beta = np.sqrt(power / np.vdot(F, F).real)
    assert relf(blk.F, F) < 1e-10
    assert abs(blk.beta - beta) / beta < 1e-10
    assert relf(blk.G, beta * F) < 1e-10


# ------------------------------------------ known answers (test_linsolve.py) --

def _rand_hpd(rng, n, cond_cap=10.0):
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    Q, _ = np.linalg.qr(A)
    P = (Q * rng.uniform(1.0, cond_cap, size=n)) @ Q.conj().T
    return (P + P.conj().T) / 2.0


@pytest.mark.gpu
def test_gpu_gs_known_answers():
    """Gauss-Seidel pins of the reference's suite (test_linsolve.py:60-96), on the GPU."""
    import paper_2305_13925_b200 as X
    from paper_2305_13925_b200.errors import ConfigurationError, SplittingError
    sysm = lambda P, s: X.HpdSystem(P=np.asarray(P, dtype=complex), rhs=np.asarray(s, dtype=complex))
    out = X.gs_solve(sysm(np.eye(3), [1.0, 2.0, 3.0]), T=1)           # identity: one sweep
    np.testing.assert_allclose(out.w, [1.0, 2.0, 3.0])
    assert out.residual_trace[-1] == 0.0
    out = X.gs_solve(sysm([[2.0, 1.0], [1.0, 2.0]], [3.0, 3.0]), T=1)  # hand-computed sweep
    np.testing.assert_allclose(out.w, [1.5, 0.75])
    rng = np.random.default_rng(2)
    for _ in range(5):                                                 # converges to direct
        P = _rand_hpd(rng, 16)
        s = rng.standard_normal(16) + 1j * rng.standard_normal(16)
        ref = np.linalg.solve(P, s)
        out = X.gs_solve(sysm(P, s), T=300)
        assert np.linalg.norm(out.w - ref) < 1e-8 * np.linalg.norm(ref)
        assert out.converged
    with pytest.raises(SplittingError):
        X.gs_solve(sysm([[0.0, 1.0], [1.0, 0.0]], [1.0, 1.0]), T=1)
    out = X.gs_solve(sysm(np.eye(2), [1.0, 1.0]), T=4)
    assert len(out.residual_trace) == out.iterations + 1
    with pytest.raises(ConfigurationError):
        X.gs_solve(sysm(np.eye(2), [1.0, 1.0]), T=0)
    P = _rand_hpd(np.random.default_rng(3), 8, 100.0)                  # eps early stop
    s = np.random.default_rng(4).standard_normal(8) + 0j
    out = X.gs_solve(sysm(P, s), T=500, eps=1e-6)
    assert out.iterations < 500 and out.converged
    assert np.sqrt(out.residual_trace[-1]) <= 1e-6


@pytest.mark.gpu
def test_gpu_jor_known_answers():
    """JOR pins of the reference's suite (test_linsolve.py:99-122), on the GPU."""
    import paper_2305_13925_b200 as X
    from paper_2305_13925_b200.errors import ConfigurationError
    sysm = lambda P, s: X.HpdSystem(P=np.asarray(P, dtype=complex), rhs=np.asarray(s, dtype=complex))
    out = X.jor_solve(sysm([[2.0, 1.0], [1.0, 2.0]], [3.0, 3.0]), T=2, omega=1.0, keep_iterates=True)
    np.testing.assert_allclose(out.iterates[0], [1.5, 1.5])
    np.testing.assert_allclose(out.iterates[1], [0.75, 0.75])
    out = X.jor_solve(sysm(np.diag([2.0, 5.0]), [4.0, 10.0]), T=1, omega=1.0)
    np.testing.assert_allclose(out.w, [2.0, 2.0])
    assert out.residual_trace[-1] == 0.0
    P = _rand_hpd(np.random.default_rng(5), 8, 100.0)                  # divergence flagged
    d = np.sqrt(np.diag(P).real)
    lam_max = np.linalg.eigvalsh(P / np.outer(d, d))[-1]
    s = np.random.default_rng(6).standard_normal(8) + 0j
    out = X.jor_solve(sysm(P, s), T=50, omega=2.5 / lam_max)
    assert not out.converged
    assert out.residual_trace[-1] > out.residual_trace[0]
    with pytest.raises(ConfigurationError):
        X.jor_solve(sysm(np.eye(2), [1.0, 1.0]), T=1, omega=0.0)
