"""Generate the committed golden fixtures from the LIVE reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``xlmimo`` from /root/reference/pkg/src (read-only, not copied),
runs the reference's own functions on seeded inputs and writes
``tests/golden/golden_*.npz``.  The fixtures pin both the CPU oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_parity.py);
neither the GPU tests nor bench.py read /root/reference at run time.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import xlmimo  # noqa: E402
from xlmimo.channel import assemble_blocks, build_correlation, psd_sqrt  # noqa: E402
from xlmimo.errors import XlMimoError  # noqa: E402
from xlmimo.linsolve import HpdSystem, cg_solve, direct_solve, gs_solve, jacpcg_solve, jor_solve  # noqa: E402
from xlmimo.metrics import sinr_eq9, sum_se  # noqa: E402
from xlmimo.precoder import BlockPrecoder, rzf_direct, rzf_iterative  # noqa: E402

from oracle.xlmimo_oracle import beta_bar, generate_channels  # noqa: E402


def random_hpd(rng, n, cond_cap=100.0):
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    Q, _ = np.linalg.qr(A)
    vals = rng.uniform(1.0, cond_cap, size=n)
    P = (Q * vals) @ Q.conj().T
    return (P + P.conj().T) / 2.0


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def sinr_adapter(H, G, sigma2):
    """Reference sinr_eq9 on one full-array block."""
    K = H.shape[1]
    K1 = K // 2
    real = assemble_blocks(np.zeros((0, K1)), H, np.zeros((0, K - K1)))
    pre = BlockPrecoder(G1=np.zeros((0, K1), complex), Gc=G,
                        G2=np.zeros((0, K - K1), complex), beta_1=0.0,
                        beta_c=0.0, beta_2=0.0, G=G)
    rep = sinr_eq9(real, pre, sigma2)
    return rep.gamma, rep.se_per_user, rep.sum_se


def solver_cases():
    """linsolve.py pins: identity RHS, vector/multi RHS, w0, eps, iterates."""
    rng = np.random.default_rng(20260101)
    out = {}
    idx = 0
    for n in (4, 8, 16, 32):
        for rep in range(2):
            P = random_hpd(rng, n, cond_cap=100.0 if rep == 0 else 1e4)
            d = np.sqrt(np.logspace(0, 3, n))
            if rep == 1:
                P = (d[:, None] * P) * d[None, :]
                P = (P + P.conj().T) / 2.0
            for rhs_kind in ("eye", "vec", "multi"):
                if rhs_kind == "eye":
                    S = np.eye(n, dtype=complex)
                elif rhs_kind == "vec":
                    S = crandn(rng, n)
                else:
                    S = crandn(rng, n, 3)
                w0 = None if rhs_kind != "multi" else 0.1 * crandn(rng, n, 3)
                T = 6
                sysm = HpdSystem(P=P, rhs=S)
                pre = f"s{idx}_"
                out[pre + "P"] = P
                out[pre + "S"] = S
                out[pre + "T"] = np.int64(T)
                if w0 is not None:
                    out[pre + "w0"] = w0
                for name, fn in (
                    ("textbook", lambda: jacpcg_solve(sysm, T, w0=w0, keep_iterates=True, variant="textbook")),
                    ("algorithm", lambda: jacpcg_solve(sysm, T, w0=w0, keep_iterates=True, variant="algorithm")),
                    ("cg", lambda: cg_solve(sysm, T, w0=w0, keep_iterates=True)),
                    ("eps", lambda: jacpcg_solve(sysm, 50, eps=1e-6, w0=w0, variant="textbook")),
                ):
                    try:
                        o = fn()
                        out[pre + name + "_w"] = o.w
                        out[pre + name + "_trace"] = o.residual_trace
                        out[pre + name + "_it"] = np.int64(o.iterations)
                        out[pre + name + "_conv"] = np.bool_(o.converged)
                        if o.iterates:
                            out[pre + name + "_iterates"] = np.stack(o.iterates)
                    except XlMimoError as exc:
                        out[pre + name + "_err"] = np.str_(type(exc).__name__)
                o = direct_solve(sysm)
                out[pre + "direct_w"] = o.w
                out[pre + "direct_trace"] = o.residual_trace
                idx += 1
    out["n_solver_cases"] = np.int64(idx)
    # error pins
    Pbad = np.diag([1.0, -1.0]).astype(complex)
    for name, fn in (
        ("direct", lambda: direct_solve(HpdSystem(P=Pbad, rhs=np.ones(2)))),
        ("cg", lambda: cg_solve(HpdSystem(P=Pbad, rhs=np.array([0.0, 1.0])), 2)),
        ("splitting", lambda: jacpcg_solve(HpdSystem(P=np.diag([0.0, 1.0]), rhs=np.ones(2)), 1)),
    ):
        try:
            fn()
            out["err_" + name] = np.str_("none")
        except XlMimoError as exc:
            out["err_" + name] = np.str_(type(exc).__name__)
    return out


def stationary_cases():
    """linsolve.py:128-176 pins: JOR (two omegas) and Gauss-Seidel on the same
    system families as solver_cases, plus their error paths."""
    rng = np.random.default_rng(20261020)
    out = {}
    idx = 0
    for n in (4, 8, 16, 32):
        for rep in range(2):
            P = random_hpd(rng, n, cond_cap=20.0 if rep == 0 else 1e3)
            if rep == 1:  # diagonally weighted: JOR/GS behave differently from the Krylov solvers
                d = np.sqrt(np.logspace(0, 2, n))
                P = (d[:, None] * P) * d[None, :]
                P = (P + P.conj().T) / 2.0
            for rhs_kind in ("eye", "vec", "multi"):
                S = np.eye(n, dtype=complex) if rhs_kind == "eye" else (
                    crandn(rng, n) if rhs_kind == "vec" else crandn(rng, n, 3))
                w0 = None if rhs_kind != "multi" else 0.1 * crandn(rng, n, 3)
                T = 6
                sysm = HpdSystem(P=P, rhs=S)
                pre = f"s{idx}_"
                out[pre + "P"] = P
                out[pre + "S"] = S
                out[pre + "T"] = np.int64(T)
                if w0 is not None:
                    out[pre + "w0"] = w0
                for name, fn in (
                    ("jor05", lambda: jor_solve(sysm, T, omega=0.5, w0=w0, keep_iterates=True)),
                    ("jor10", lambda: jor_solve(sysm, T, omega=1.0, w0=w0, keep_iterates=True)),
                    ("gs", lambda: gs_solve(sysm, T, w0=w0, keep_iterates=True)),
                    ("gseps", lambda: gs_solve(sysm, 40, w0=w0, eps=1e-5)),
                ):
                    o = fn()
                    out[pre + name + "_w"] = o.w
                    out[pre + name + "_trace"] = o.residual_trace
                    out[pre + name + "_it"] = np.int64(o.iterations)
                    out[pre + name + "_conv"] = np.bool_(o.converged)
                    if o.iterates:
                        out[pre + name + "_iterates"] = np.stack(o.iterates)
                idx += 1
    out["n_cases"] = np.int64(idx)
    for name, fn in (
        ("gs_zero_diag", lambda: gs_solve(HpdSystem(P=np.diag([0.0, 1.0]), rhs=np.ones(2)), 1)),
        ("jor_zero_diag", lambda: jor_solve(HpdSystem(P=np.diag([1.0, 0.0]), rhs=np.ones(2)), 1)),
        ("jor_omega", lambda: jor_solve(HpdSystem(P=np.eye(2), rhs=np.ones(2)), 1, omega=0.0)),
        ("gs_T0", lambda: gs_solve(HpdSystem(P=np.eye(2), rhs=np.ones(2)), 0)),
    ):
        try:
            fn()
            out["err_" + name] = np.str_("none")
        except XlMimoError as exc:
            out["err_" + name] = np.str_(type(exc).__name__)
    return out


def telemetry_cases():
    """metrics.py:93-185 pins.

    convergence_trace: the reference function itself on its default
    configuration (trials = 6, T_max = 8), plus the central-subarray channel
    Hc and QPSK right-hand side of every trial, extracted with the same
    seed_stream / draw_trial sequence the function uses.
    ber_montecarlo: one SNR point's inner loop, made of the reference's own
    functions (draw_trial, _precoders_for_trial, coupling_matrix,
    qpsk_modulate, qpsk_detect): coupling matrices, bits, noise and the error
    counts, plus the reference function's own report for the same settings.
    """
    from xlmimo.config import ExperimentConfig
    from xlmimo.metrics import (_precoders_for_trial, ber_montecarlo, convergence_trace,
                                coupling_matrix, qpsk_detect, qpsk_modulate)
    from xlmimo.scenario import build_scenario, draw_trial
    from xlmimo.seeding import seed_stream

    out = {}
    cfg = ExperimentConfig()
    cfg.run.trials, cfg.run.t_max = 6, 8
    methods = ["gs", "jor", "cg", "jacpcg"]
    med = convergence_trace(cfg, methods=methods)
    scen = build_scenario(cfg)
    Hc, S = [], []
    for trial in range(cfg.run.trials):
        rng = seed_stream(cfg.run.seed, trial)
        draw = draw_trial(scen, rng)
        bits = rng.integers(0, 2, size=(scen.K, 2), dtype=np.int8)
        Hc.append(draw.realization.Hc)
        S.append(qpsk_modulate(bits))
    out["conv_Hc"] = np.stack(Hc)
    out["conv_S"] = np.stack(S)
    out["conv_xi"] = np.float64(cfg.power.xi)
    out["conv_omega"] = np.float64(cfg.solver.omega)
    out["conv_variant"] = np.str_(cfg.solver.pcg_variant)
    out["conv_T"] = np.int64(cfg.run.t_max)
    out["conv_methods"] = np.array(methods)
    for m in methods:
        out["conv_median_" + m] = med[m]

    # BER: one grid point, the reference's loop body (metrics.py:124-140)
    cfg = ExperimentConfig()
    cfg.run.symbols_per_channel = 64
    nsym = cfg.run.symbols_per_channel
    grid = np.array([4.0, 10.0])
    bmethods = ["direct", "jacpcg", "jor"]
    scen = build_scenario(cfg)
    K = scen.K
    cfg.run.bits_per_point = 3 * 2 * K * nsym  # three channel draws per point
    rep = ber_montecarlo(cfg, bmethods, snr_grid_db=grid)
    sigma2 = cfg.power.sigma2_watts
    for ig, snr_db in enumerate(grid):
        snr = 10.0 ** (snr_db / 10.0)
        xi, power = 1.0 / snr, sigma2 * snr
        for trial in range(3):
            rng = seed_stream(cfg.run.seed, trial * grid.size + ig)
            draw = draw_trial(scen, rng)
            pre = _precoders_for_trial(draw.realization, xi, power, bmethods, cfg.solver.T,
                                       cfg.solver.omega, cfg.solver.pcg_variant)
            bits = rng.integers(0, 2, size=(K, nsym, 2), dtype=np.int8)
            noise = np.sqrt(sigma2 / 2.0) * (rng.standard_normal((K, nsym))
                                             + 1j * rng.standard_normal((K, nsym)))
            key = f"ber_p{ig}_t{trial}_"
            out[key + "bits"] = bits
            out[key + "noise"] = noise
            out[key + "H"] = draw.realization.H
            for m in bmethods:
                Bm = coupling_matrix(draw.realization, pre[m])
                gain = np.diag(Bm).copy()
                gain[gain == 0] = 1.0
                Y = Bm @ qpsk_modulate(bits) + noise
                out[key + m + "_B"] = Bm
                out[key + m + "_G"] = pre[m].G
                out[key + m + "_errors"] = np.int64(np.count_nonzero(qpsk_detect(Y / gain[:, None]) != bits))
    out["ber_grid"] = grid
    out["ber_methods"] = np.array(bmethods)
    out["ber_nsym"] = np.int64(nsym)
    out["ber_sigma2"] = np.float64(sigma2)
    for m in bmethods:
        out["ber_report_errors_" + m] = rep.bit_errors[m]
    out["ber_report_bits"] = np.int64(rep.bits_simulated)
    return out


def block_cases():
    """precoder.py:118-146 + metrics.py:35-58 pins for the S=3/L=2 block
    topology: the reference's own draws (default
    configuration), build_precoder for every method with per-block beta, and
    sinr_eq9 on the block coupling."""
    from xlmimo.config import ExperimentConfig
    from xlmimo.precoder import build_precoder
    from xlmimo.scenario import build_scenario, draw_trial
    from xlmimo.seeding import seed_stream

    cfg = ExperimentConfig()
    scen = build_scenario(cfg)
    xi, power, sigma2 = cfg.power.xi, cfg.power.tx_power_watts, cfg.power.sigma2_watts
    methods = ["direct", "jacpcg", "cg", "jor", "gs"]
    out = {"xi": np.float64(xi), "power": np.float64(power), "sigma2": np.float64(sigma2),
           "T": np.int64(cfg.solver.T), "omega": np.float64(cfg.solver.omega),
           "variant": np.str_(cfg.solver.pcg_variant), "methods": np.array(methods)}
    n = 0
    for trial in range(8):
        draw = draw_trial(scen, seed_stream(cfg.run.seed, trial))
        r = draw.realization
        key = f"r{trial}_"
        out[key + "H1"], out[key + "Hc"], out[key + "H2"], out[key + "H"] = r.H1, r.Hc, r.H2, r.H
        for m in methods:
            bp = build_precoder(r, xi, power, m, T=cfg.solver.T, omega=cfg.solver.omega,
                                pcg_variant=cfg.solver.pcg_variant)
            rep = sinr_eq9(r, bp, sigma2)
            out[key + m + "_G"] = bp.G
            out[key + m + "_betas"] = np.array([bp.beta_1, bp.beta_c, bp.beta_2])
            out[key + m + "_gamma"] = rep.gamma
            out[key + m + "_sumse"] = np.float64(rep.sum_se)
        n += 1
    out["n"] = np.int64(n)
    return out


def precoder_cases():
    """precoder.py / metrics.py pins on BASELINE-model and random channels."""
    out = {}
    cases = [
        # (tag, H batch)
        ("cfg1", generate_channels(0, 0, 2, 4, 16, 0.5, 0.5)),      # M=256,K=16
        ("small", generate_channels(7, 100, 4, 1, 8, 0.5, 0.7)),    # M=64,K=8
        ("rand", np.stack([crandn(np.random.default_rng(5 + i), 48, 12) for i in range(3)])),
    ]
    snr = 10.0
    for tag, Hb in cases:
        B, M, K = Hb.shape
        P_tx = 10 ** (snr / 10)
        alpha = K / P_tx
        sigma2 = 1.0
        out[tag + "_H"] = Hb
        out[tag + "_alpha"] = np.float64(alpha)
        out[tag + "_power"] = np.float64(P_tx)
        out[tag + "_sigma2"] = np.float64(sigma2)
        for meth in ("jacpcg_textbook", "jacpcg_algorithm", "cg", "direct"):
            for T in ((4,) if tag == "cfg1" else (1, 4)):
                if meth == "direct" and T != 4:
                    continue
                Gs, Fs, betas, gams, ses = [], [], [], [], []
                for b in range(B):
                    H = Hb[b]
                    if meth == "direct":
                        blk = rzf_direct(H, alpha, P_tx)
                    elif meth == "cg":
                        blk = rzf_iterative(H, alpha, P_tx, solver="cg", T=T)
                    else:
                        blk = rzf_iterative(H, alpha, P_tx, solver="jacpcg", T=T,
                                            pcg_variant=meth.split("_")[1])
                    g, _, s = sinr_adapter(H, blk.G, sigma2)
                    Gs.append(blk.G)
                    Fs.append(blk.F)
                    betas.append(blk.beta)
                    gams.append(g)
                    ses.append(s)
                key = f"{tag}_{meth}_T{T}"
                out[key + "_G"] = np.stack(Gs)
                out[key + "_beta"] = np.array(betas)
                out[key + "_gamma"] = np.stack(gams)
                out[key + "_sumse"] = np.array(ses)
        out[tag + "_gram"] = np.stack([xlmimo.gram_regularized(H, alpha).P for H in Hb])
    # analytic pins (test_precoder.py:14-63)
    out["gram_zero"] = xlmimo.gram_regularized(np.zeros((4, 3)), 0.5).P
    out["gram_eye"] = xlmimo.gram_regularized(np.eye(2), 1.0).P
    blk = rzf_direct(np.eye(2), 1.0, 3.0)
    out["direct_eye_F"] = blk.F
    out["direct_eye_beta"] = np.float64(blk.beta)
    try:
        rzf_direct(np.zeros((4, 2)), 0.5, 1.0)
        out["err_degenerate"] = np.str_("none")
    except XlMimoError as exc:
        out["err_degenerate"] = np.str_(type(exc).__name__)
    # sum_se pins
    trials = np.random.default_rng(3).uniform(10, 20, size=37)
    m, s = sum_se(trials)
    out["sumse_in"] = trials
    out["sumse_mean"] = np.float64(m)
    out["sumse_sem"] = np.float64(s)
    return out


def channel_cases():
    """channel.py:33-53 correlation square roots and flops.py integers."""
    out = {}
    for r in (0.5, 0.7, 0.9):
        out[f"rsqrt_{r}"] = psd_sqrt(build_correlation(64, r))
    out["beta_bar"] = np.float64(beta_bar())
    flops = {}
    for K in (1, 16, 30, 64, 128, 256):
        flops[f"direct_{K}"] = xlmimo.flops_direct(K)
        for T in (1, 4, 5, 6):
            flops[f"cg_{K}_{T}"] = xlmimo.flops_cg(K, T)
            flops[f"jacpcg_{K}_{T}"] = xlmimo.flops_jacpcg(K, T)
    out["flops_keys"] = np.array(list(flops.keys()))
    out["flops_vals"] = np.array(list(flops.values()), dtype=np.int64)
    return out


FIXTURES = {
    "solvers": solver_cases,
    "precoders": precoder_cases,
    "channel": channel_cases,
    "stationary": stationary_cases,
    "telemetry": telemetry_cases,
    "blocks": block_cases,
}


def main(names=None):
    """python tests/golden/make_golden.py [fixture ...]  (default: all)"""
    for name in names or FIXTURES:
        np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"), **FIXTURES[name]())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main(sys.argv[1:])
