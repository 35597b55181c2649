"""Convergence telemetry and the BER chain (metrics.py:93-185).

Fixtures: tests/golden/golden_telemetry.npz, written by make_golden.py from the
reference's own convergence_trace (default configuration, 6 trials, T_max = 8)
and from one SNR point of ber_montecarlo's loop body (its own draw_trial,
_precoders_for_trial, coupling_matrix, qpsk_modulate, qpsk_detect).
"""

import numpy as np
import pytest

from oracle import xlmimo_oracle as O


def _oracle_trace(P, s, m, T, omega, variant):
    if m == "gs":
        o = O.gs_solve(P, s, T)
    elif m == "jor":
        o = O.jor_solve(P, s, T, omega=omega)
    elif m == "cg":
        o = O.cg_solve(P, s, T)
    else:
        o = O.jacpcg_solve(P, s, T, variant=variant)
    tr = np.empty(T + 1)
    tr[: o.residual_trace.size] = o.residual_trace
    tr[o.residual_trace.size:] = o.residual_trace[-1]
    return tr


def test_oracle_convergence_median_golden(golden):
    """The oracle's solvers + the reference's padding + np.median reproduce the
    reference's convergence_trace (pins the oracle for this row)."""
    g = golden("telemetry")
    T, xi, omega, var = int(g["conv_T"]), float(g["conv_xi"]), float(g["conv_omega"]), str(g["conv_variant"])
    for m in g["conv_methods"]:
        traces = np.stack([_oracle_trace(O.gram_regularized(Hc, xi), s, str(m), T, omega, var)
                           for Hc, s in zip(g["conv_Hc"], g["conv_S"])])
        np.testing.assert_allclose(np.median(traces, axis=0), g["conv_median_" + str(m)], rtol=1e-9, atol=1e-15)


def _np_errors(Bm, bits, noise):
    gain = np.diag(Bm).copy()
    gain[gain == 0] = 1.0
    s = ((1.0 - 2.0 * bits[..., 0]) + 1j * (1.0 - 2.0 * bits[..., 1])) / np.sqrt(2.0)
    Y = Bm @ s + noise
    z = Y / gain[:, None]
    det = np.stack([(z.real < 0).astype(np.int8), (z.imag < 0).astype(np.int8)], axis=-1)
    return int(np.count_nonzero(det != bits))


def _ber_keys(g):
    for ig in range(len(g["ber_grid"])):
        for t in range(3):
            for m in g["ber_methods"]:
                yield ig, t, str(m), f"ber_p{ig}_t{t}_"


def test_ber_fixture_consistency(golden):
    g = golden("telemetry")
    tot = {}
    for ig, t, m, key in _ber_keys(g):
        e = _np_errors(g[key + m + "_B"], g[key + "bits"], g[key + "noise"])
        assert e == int(g[key + m + "_errors"])
        tot[(m, ig)] = tot.get((m, ig), 0) + e
    for m in g["ber_methods"]:
        m = str(m)
        np.testing.assert_array_equal([tot[(m, ig)] for ig in range(len(g["ber_grid"]))],
                                      g["ber_report_errors_" + m])


# ------------------------------------------------------------------ GPU -----

@pytest.mark.gpu
def test_gpu_convergence_median_golden(golden):
    import torch
    from paper_2305_13925_b200 import telemetry as TM
    g = golden("telemetry")
    H = torch.from_numpy(g["conv_Hc"]).cuda()
    S = torch.from_numpy(g["conv_S"]).cuda()
    tr = TM.convergence_traces_batched(H, float(g["conv_xi"]), S, [str(m) for m in g["conv_methods"]],
                                       int(g["conv_T"]), omega=float(g["conv_omega"]),
                                       variant=str(g["conv_variant"]))
    for m in g["conv_methods"]:
        np.testing.assert_allclose(TM.median_trace(tr[str(m)]), g["conv_median_" + str(m)],
                                   rtol=1e-7, atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_gpu_ber_errors_golden(golden, dt):
    """xl_ber_errors on the reference's coupling matrices, bits and noise: the
    bit-error counts are integers and must match exactly in complex128; the
    complex64 chain may flip decisions only where |Re|, |Im| of Y/gain sit
    within fp32 round-off of zero."""
    import torch
    from paper_2305_13925_b200 import telemetry as TM
    g = golden("telemetry")
    cdt = torch.complex128 if dt == "c128" else torch.complex64
    keys = list(_ber_keys(g))
    Bc = torch.stack([torch.from_numpy(g[k + m + "_B"]) for _, _, m, k in keys]).to("cuda", cdt)
    bits = torch.stack([torch.from_numpy(g[k + "bits"]) for _, _, m, k in keys]).cuda()
    noise = torch.stack([torch.from_numpy(g[k + "noise"]) for _, _, m, k in keys]).to("cuda", cdt)
    err = TM.ber_errors_batched(Bc, bits, noise).cpu().numpy()
    ref = np.array([int(g[k + m + "_errors"]) for _, _, m, k in keys])
    if dt == "c128":
        np.testing.assert_array_equal(err, ref)
    else:
        assert np.abs(err - ref).max() <= 2, (err, ref)


@pytest.mark.gpu
def test_gpu_block_coupling_golden(golden):
    """coupling of the reference's three-block precoders through the device
    coupling (stacked block matrices give the block coupling, test_metrics.py:39-44)."""
    import torch
    from paper_2305_13925_b200 import batched as BT
    g = golden("telemetry")
    for _, _, m, k in _ber_keys(g):
        H = torch.from_numpy(g[k + "H"])[None].cuda()
        G = torch.from_numpy(g[k + m + "_G"])[None].cuda()
        B = BT.sinr_batched(H, G, 1.0).coupling[0].cpu().numpy()
        ref = g[k + m + "_B"]
        assert np.linalg.norm(B - ref) / np.linalg.norm(ref) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["direct", "jacpcg", "jor"])
def test_gpu_ber_point_vs_oracle(method):
    """ber_point_batched end to end (single-block precoders) against the oracle
    precoder + the numpy chain on the same draws: identical error counts."""
    import torch
    import paper_2305_13925_b200 as X
    from paper_2305_13925_b200 import telemetry as TM
    rng = np.random.default_rng(11)
    B, M, K, nsym = 6, 64, 8, 128
    m = X.ChannelModel(S=1, K=K, p=0.5, r=0.7)
    H = X.generate_channels(m, seed=2, first=0, B=B, dtype=torch.complex128)
    xi, power, sigma2 = 0.5, 4.0, 1.0
    bits = rng.integers(0, 2, size=(B, K, nsym, 2), dtype=np.int8)
    noise = np.sqrt(sigma2 / 2) * (rng.standard_normal((B, K, nsym)) + 1j * rng.standard_normal((B, K, nsym)))
    got = TM.ber_point_batched(H, xi, power, [method], torch.from_numpy(bits), torch.from_numpy(noise).cuda(),
                               T=4, omega=0.8)[method].cpu().numpy()
    Hn = H.cpu().numpy()
    for b in range(B):
        P = O.gram_regularized(Hn[b], xi)
        if method == "direct":
            Xs = O.direct_solve(P, np.eye(K)).w
        elif method == "jacpcg":
            Xs = O.jacpcg_solve(P, np.eye(K), 4, variant="textbook").w
        else:
            Xs = O.jor_solve(P, np.eye(K), 4, omega=0.8).w
        F = Hn[b] @ Xs
        G = np.sqrt(power / np.vdot(F, F).real) * F
        assert got[b] == _np_errors(Hn[b].conj().T @ G, bits[b], noise[b]), b


# ------------------------------------------------------- block topology -----

def test_oracle_blocks_golden(golden):
    """Oracle per-block RZF + stacked coupling reproduce the reference's
    build_precoder / sinr_eq9 on its own draws (pins the oracle for next-2)."""
    g = golden("blocks")
    xi, power, sigma2, T, omega = (float(g["xi"]), float(g["power"]), float(g["sigma2"]),
                                   int(g["T"]), float(g["omega"]))
    for t in range(int(g["n"])):
        k = f"r{t}_"
        H1, Hc, H2, H = g[k + "H1"], g[k + "Hc"], g[k + "H2"], g[k + "H"]
        for m in g["methods"]:
            m = str(m)
            Gs, betas = [], []
            for Hb in (H1, Hc, H2):
                P = O.gram_regularized(Hb, xi)
                Kb = Hb.shape[1]
                Xs = {"direct": lambda: O.direct_solve(P, np.eye(Kb)).w,
                      "jacpcg": lambda: O.jacpcg_solve(P, np.eye(Kb), T, variant=str(g["variant"])).w,
                      "cg": lambda: O.cg_solve(P, np.eye(Kb), T).w,
                      "jor": lambda: O.jor_solve(P, np.eye(Kb), T, omega=omega).w,
                      "gs": lambda: O.gs_solve(P, np.eye(Kb), T).w}[m]()
                F = Hb @ Xs
                beta = np.sqrt(power / np.vdot(F, F).real)
                Gs.append(beta * F)
                betas.append(beta)
            K1 = H1.shape[1]
            G = np.zeros_like(H)
            G[:H1.shape[0], :K1] = Gs[0]
            G[H1.shape[0]:H1.shape[0] + Hc.shape[0]] = Gs[1]
            G[H1.shape[0] + Hc.shape[0]:, K1:] = Gs[2]
            assert np.linalg.norm(G - g[k + m + "_G"]) / np.linalg.norm(g[k + m + "_G"]) < 1e-10, (t, m)
            np.testing.assert_allclose(betas, g[k + m + "_betas"], rtol=1e-10)
            gam, _, s = O.sinr_single_block(H, G, sigma2)
            np.testing.assert_allclose(gam, g[k + m + "_gamma"], rtol=1e-8)
            assert abs(s - float(g[k + m + "_sumse"])) < 1e-9 * abs(s)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_gpu_block_precoder_golden(golden, dt):
    """build_precoder_batched + block_sinr_batched on the reference's draws
    (all 8 in one batch) against the reference's block precoders and SINR."""
    import torch
    from paper_2305_13925_b200 import blocks as BK
    g = golden("blocks")
    cdt = torch.complex128 if dt == "c128" else torch.complex64
    n = int(g["n"])
    stack = lambda name: torch.stack([torch.from_numpy(g[f"r{t}_{name}"]) for t in range(n)]).to("cuda", cdt)
    H1, Hc, H2 = stack("H1"), stack("Hc"), stack("H2")
    xi, power, sigma2 = float(g["xi"]), float(g["power"]), float(g["sigma2"])
    tol_g = 1e-10 if dt == "c128" else 1e-4
    for m in g["methods"]:
        m = str(m)
        pre = BK.build_precoder_batched(H1, Hc, H2, xi, power, m, T=int(g["T"]), omega=float(g["omega"]),
                                        variant=str(g["variant"]))
        rep = BK.block_sinr_batched(H1, Hc, H2, pre, sigma2)
        G = pre.G.cpu().numpy()
        betas = torch.stack([pre.beta_1, pre.beta_c, pre.beta_2], 1).cpu().numpy()
        for t in range(n):
            ref = g[f"r{t}_{m}_G"]
            assert np.linalg.norm(G[t] - ref) / np.linalg.norm(ref) < tol_g, (m, t)
            np.testing.assert_allclose(betas[t], g[f"r{t}_{m}_betas"], rtol=10 * tol_g)
            np.testing.assert_allclose(rep.gamma[t].cpu().numpy(), g[f"r{t}_{m}_gamma"], rtol=100 * tol_g)
            assert abs(rep.sum_se[t].item() - float(g[f"r{t}_{m}_sumse"])) < 10 * tol_g * float(g[f"r{t}_{m}_sumse"])
