"""Pin the CPU oracle (oracle/xlmimo_oracle.py) to the reference's own outputs.

The fixtures were written by tests/golden/make_golden.py from the live
reference package; this file runs on CPU only.
"""

import numpy as np
import pytest

from oracle import xlmimo_oracle as O


def test_solver_golden(golden):
    g = golden("solvers")
    n = int(g["n_solver_cases"])
    assert n == 24
    for i in range(n):
        pre = f"s{i}_"
        P, S, T = g[pre + "P"], g[pre + "S"], int(g[pre + "T"])
        w0 = g[pre + "w0"] if pre + "w0" in g else None
        runs = {
            "textbook": lambda: O.jacpcg_solve(P, S, T, w0=w0, keep_iterates=True, variant="textbook"),
            "algorithm": lambda: O.jacpcg_solve(P, S, T, w0=w0, keep_iterates=True, variant="algorithm"),
            "cg": lambda: O.cg_solve(P, S, T, w0=w0, keep_iterates=True),
            "eps": lambda: O.jacpcg_solve(P, S, 50, eps=1e-6, w0=w0, variant="textbook"),
        }
        for name, fn in runs.items():
            if pre + name + "_err" in g:
                with pytest.raises(O.OracleError) as ei:
                    fn()
                assert ei.value.kind == str(g[pre + name + "_err"])
                continue
            o = fn()
            # same numpy operations in the same order as the reference
            np.testing.assert_array_equal(o.w, g[pre + name + "_w"])
            np.testing.assert_array_equal(o.residual_trace, g[pre + name + "_trace"])
            assert o.iterations == int(g[pre + name + "_it"])
            assert o.converged == bool(g[pre + name + "_conv"])
            if pre + name + "_iterates" in g:
                np.testing.assert_array_equal(np.stack(o.iterates), g[pre + name + "_iterates"])
        o = O.direct_solve(P, S)
        np.testing.assert_allclose(o.w, g[pre + "direct_w"], rtol=0, atol=1e-13 * np.abs(g[pre + "direct_w"]).max())


def test_solver_error_kinds(golden):
    g = golden("solvers")
    Pbad = np.diag([1.0, -1.0]).astype(complex)
    with pytest.raises(O.OracleError) as e1:
        O.direct_solve(Pbad, np.ones(2))
    assert e1.value.kind == str(g["err_direct"])
    with pytest.raises(O.OracleError) as e2:
        O.cg_solve(Pbad, np.array([0.0, 1.0]), 2)
    assert e2.value.kind == str(g["err_cg"])
    with pytest.raises(O.OracleError) as e3:
        O.jacpcg_solve(np.diag([0.0, 1.0]), np.ones(2), 1)
    assert e3.value.kind == str(g["err_splitting"])


@pytest.mark.parametrize("tag", ["cfg1", "small", "rand"])
def test_precoder_golden(golden, tag):
    g = golden("precoders")
    Hb = g[tag + "_H"]
    alpha, power, sigma2 = float(g[tag + "_alpha"]), float(g[tag + "_power"]), float(g[tag + "_sigma2"])
    for b in range(Hb.shape[0]):
        np.testing.assert_array_equal(O.gram_regularized(Hb[b], alpha), g[tag + "_gram"][b])
    for key in [k for k in g.files if k.startswith(tag + "_") and k.endswith("_G")]:
        meth_T = key[len(tag) + 1:-2]
        meth, T = meth_T.rsplit("_T", 1)
        T = int(T)
        for b in range(Hb.shape[0]):
            if meth == "direct":
                G, _, beta = O.rzf_direct(Hb[b], alpha, power)
            elif meth == "cg":
                G, _, beta = O.rzf_iterative(Hb[b], alpha, power, "cg", T)
            else:
                G, _, beta = O.rzf_iterative(Hb[b], alpha, power, "jacpcg", T,
                                             pcg_variant=meth.split("_")[1])
            ref = g[key][b]
            err = np.linalg.norm(G - ref) / np.linalg.norm(ref)
            assert err <= 1e-13, (key, b, err)
            assert beta == pytest.approx(g[key[:-2] + "_beta"][b], rel=1e-13)
            gamma, _, s = O.sinr_single_block(Hb[b], ref, sigma2)
            np.testing.assert_allclose(gamma, g[key[:-2] + "_gamma"][b], rtol=1e-12)
            assert s == pytest.approx(g[key[:-2] + "_sumse"][b], rel=1e-13)


def test_analytic_pins(golden):
    g = golden("precoders")
    np.testing.assert_array_equal(O.gram_regularized(np.zeros((4, 3)), 0.5), g["gram_zero"])
    np.testing.assert_array_equal(O.gram_regularized(np.eye(2), 1.0), g["gram_eye"])
    G, F, beta = O.rzf_direct(np.eye(2), 1.0, 3.0)
    np.testing.assert_allclose(F, g["direct_eye_F"], atol=1e-15)
    assert beta == pytest.approx(float(g["direct_eye_beta"]))
    with pytest.raises(O.OracleError) as ei:
        O.rzf_direct(np.zeros((4, 2)), 0.5, 1.0)
    assert ei.value.kind == str(g["err_degenerate"])
    m, s = O.sum_se(g["sumse_in"])
    assert m == float(g["sumse_mean"]) and s == float(g["sumse_sem"])


def test_channel_and_flops_golden(golden):
    g = golden("channel")
    for r in (0.5, 0.7, 0.9):
        np.testing.assert_allclose(O.correlation_sqrt(64, r), g[f"rsqrt_{r}"], rtol=0, atol=1e-13)
    assert O.beta_bar() == pytest.approx(2.0611e-9, rel=1e-4)
    assert O.beta_bar() == float(g["beta_bar"])
    for k, v in zip(g["flops_keys"], g["flops_vals"]):
        parts = str(k).split("_")
        if parts[0] == "direct":
            assert O.flops_direct(int(parts[1])) == v
        elif parts[0] == "cg":
            assert O.flops_cg(int(parts[1]), int(parts[2])) == v
        else:
            assert O.flops_jacpcg(int(parts[1]), int(parts[2])) == v
    # the paper's published pins (test_flops.py:11-49)
    assert O.flops_direct(30) == 108029 and O.flops_jacpcg(30, 5) == 46530


def test_philox_known_answer():
    """Random123 Philox4x32-10 known-answer vectors (kat_vectors)."""
    out = O.philox4x32_10(0, 0, 0, 0, 0, 0)
    assert [int(x) for x in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    out = O.philox4x32_10(0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF)
    assert [int(x) for x in out] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    out = O.philox4x32_10(0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0)
    assert [int(x) for x in out] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_channel_statistics():
    """Generator pins in the style of test_channel.py:152-173."""
    S, K, p, r = 4, 8, 0.5, 0.5
    H = O.generate_channels(11, 0, 400, S, K, p, r)
    assert H.shape == (400, 256, K)
    blocks = H.reshape(400, S, 64, K)
    energy = (np.abs(blocks) ** 2).sum(axis=2)           # (B, S, K)
    vis = energy > 0
    assert vis.any(axis=1).all()                          # >= 1 visible subarray per user
    # invisible subarrays are exact zeros; visible fraction ~ p / (1 - (1-p)^S)
    frac = vis.mean()
    assert abs(frac - p / (1 - (1 - p) ** S)) < 0.03
    # within a visible block: covariance ~ gain * R (3% Frobenius over many draws)
    Rs = O.correlation_sqrt(64, r)
    R = Rs @ Rs
    Hn, amp, _ = O.generate_channels(12, 0, 16000, 1, 4, 1.0, r, return_parts=True)
    z = Hn / amp[:, None, :]
    emp = np.einsum("bik,bjk->ij", z, z.conj()) / (z.shape[0] * z.shape[2])
    assert np.linalg.norm(emp - R) / np.linalg.norm(R) < 0.03
    # determinism and index addressing: a sub-range reproduces the full batch
    H2 = O.generate_channels(11, 100, 50, S, K, p, r)
    np.testing.assert_array_equal(H2, H[100:150])
