"""Benchmark: Jac-PCG RZF precoders/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

A step = one pass of the hot path over one batch resident in HBM: the fused
precoder (Gram -> Jac-PCG T iterations -> beta, W -> SINR/SE) for B
realizations, plus the ergodic-SE partials (and their NCCL all-gather when
N > 1).  Weak scaling: every rank owns B realizations of its own index range.

Prints ONE JSON line on rank 0 (contract in the task statement):
value = precoders/s of the whole job (device-timed, CUDA events, max over
ranks), e2e = the same metric through the host-buffer API (pinned H in, W and
SE out, copies inside the timed region), roofline of the fused precoder call,
cpu_baseline = the CPU oracle port on this host's cores (rank 0, N = 1).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Jac-PCG RZF precoders/sec (batched MxK)"
UNIT = "precoders/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--batch", type=int, default=None, help="realizations per rank per step")
    ap.add_argument("--method", default="jacpcg")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=256,
                    help="realizations per HostPipeline chunk (fill/drain ~ 1/number of chunks)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------- helpers ----

def flops_per_precoder(M, K, T, method):
    """Algorithmic real flops per precoder (flops.py:35-69)."""
    from oracle.xlmimo_oracle import flops_cg, flops_direct, flops_jacpcg
    if method == "jacpcg":
        solve = K * flops_jacpcg(K, T)
    elif method == "cg":
        solve = K * flops_cg(K, T)
    else:
        solve = flops_direct(K)
    return 4 * M * K * (K + 1) + solve + 8 * M * K * K + 8 * K ** 3


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6551.7), d.get("bf16_tflops", 1640.2), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during timing."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.limit_w = None
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "power_limit_w": self.limit_w,
                "samples": len(self.samples)}


# ------------------------------------------------------ CPU oracle baseline --

def _cpu_worker(args):
    """One host core: oracle precoder + SE on pre-generated H for ~seconds."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    seconds, cfg_name, method, seed, first, B = args
    sys.path.insert(0, ROOT)
    import numpy as np  # noqa: F401
    from oracle import xlmimo_oracle as O
    from paper_2305_13925_b200.configs import CONFIGS
    wl = CONFIGS[cfg_name]
    m = wl.model
    H = O.generate_channels(seed, first, B, m.S, m.K, m.p, m.r, Ms=m.Ms)
    done, t0 = 0, time.perf_counter()
    while True:
        O.precoder_and_se(H[done % B], wl.alpha(), wl.power(), 1.0, method, wl.T, "textbook")
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return done, el


def cpu_baseline(cfg_name, method, seconds):
    """Oracle port on all host cores (ProcessPool, BLAS pinned to 1 thread: F7)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    ctx = mp.get_context("spawn")
    with cf.ProcessPoolExecutor(cores, mp_context=ctx) as ex:
        res = list(ex.map(_cpu_worker, [(seconds, cfg_name, method, 7, 10_000 + 16 * i, 16)
                                        for i in range(cores)]))
        # also one core alone (the rest of the pool idle)
        n1, el1 = ex.submit(_cpu_worker, (min(4.0, seconds), cfg_name, method, 7, 10_000, 16)).result()
    n = sum(r[0] for r in res)
    el = max(r[1] for r in res)
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "")
    except OSError:
        pass
    return {"value": n / el, "unit": UNIT, "cores": cores, "kind": "port",
            "single_core_value": n1 / el1, "cpu_model": model,
            "sample": f"{n} {cfg_name} precoders ({method}, T={_T(cfg_name)}) + SINR/SE, "
                      f"complex128 oracle, {cores} processes x 1 BLAS thread, {el:.1f} s"}


def _T(cfg_name):
    from paper_2305_13925_b200.configs import CONFIGS
    return CONFIGS[cfg_name].T


# ------------------------------------------------------------------ main ----

def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2305_13925_b200.configs import CONFIGS
    wl = CONFIGS[a.config]
    secs = max(2.0, min(a.cpu_seconds, 150.0 / max(1, a.steps + a.warmup)))
    vals = []
    cb = None
    for i in range(a.warmup + a.steps):
        cb = cpu_baseline(a.config, a.method, secs)
        if i >= a.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1000.0 * secs, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"{a.config}: M={wl.M}, K={wl.K}, T={wl.T}, {a.method} "
                                   f"(reference algorithm, CPU port, per-step sample of {secs:.0f} s)"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_2305_13925_b200 as X
    from paper_2305_13925_b200 import _lib as L
    from paper_2305_13925_b200 import batched as BT
    from paper_2305_13925_b200.distributed import ergodic_se

    wl = X.CONFIGS[a.config]
    M, K, T = wl.M, wl.K, wl.T
    dt = wl.dtype
    csz = 8 if dt == torch.complex64 else 16
    # cfg4 (configs[3]): 65536 realizations over all GPUs, generated on device in
    # chunks of 2048 per GPU inside the step (they do not fit HBM at once: 256 GiB);
    # other configs: the rank's batch is resident in HBM, precoded in sub-batches
    # of at most 16 GiB of H (cfg5: 4 x 2048)
    gen_in_step = wl.chunk is not None
    if gen_in_step:
        B = a.batch or wl.B // world
        sub = min(wl.chunk, B)
    else:
        B = a.batch or wl.B
        sub = B if B * M * K * csz <= 16 * 2**30 else 2048
    assert B % sub == 0, "batch must be a multiple of the sub-batch"
    first = rank * B
    alpha, power = wl.alpha(), wl.power()
    lib = L.lib()
    tc = X.uses_tensor_cores(dt, a.method, M, K)
    H = X.generate_channels(wl.model, seed=0, first=first, B=sub if gen_in_step else B, dtype=dt, device=dev)
    out = BT.alloc_outputs(H[:sub], want_gamma=True)
    se_all = torch.empty(B, dtype=torch.float64, device=dev)
    st_all = torch.empty(B, dtype=torch.int32, device=dev)

    def step(record=None):
        for c0 in range(0, B, sub):
            if gen_in_step:
                X.generate_channels(wl.model, seed=0, first=first + c0, B=sub, dtype=dt, device=dev, out=H,
                                    check=False)
                Hc = H
            else:
                Hc = H[c0:c0 + sub]
            if record is not None:
                record[c0 // sub][0].record()
            BT.rzf_batched(Hc, alpha, power, method=a.method, T=T, variant="textbook", sigma2=1.0,
                           out=out, check=False)
            if record is not None:
                record[c0 // sub][1].record()
            if sub < B:
                se_all[c0:c0 + sub].copy_(out.sum_se)
                st_all[c0:c0 + sub].copy_(out.status)
        return ergodic_se(out.sum_se if sub == B else se_all, chunk=2048, group=None if world > 1 else False)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    L.raise_status((out.status if sub == B else st_all).cpu().numpy(), "bench warm-up")

    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(B // sub)] for _ in range(a.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = lib.xl_launch_count()
    with ClockSampler(local) as clk:
        t0.record()
        for i in range(a.steps):
            se_mean = step(ev[i])
        t1.record()
        torch.cuda.synchronize()
    launches = int(lib.xl_launch_count() - n0)
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    # the precoder calls of one step (without the in-step channel generation)
    kern_ms = statistics.mean(sum(e0.elapsed_time(e1) for e0, e1 in evs) for evs in ev)
    if world > 1:
        tt = torch.tensor([ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, kern_ms = float(tt[0]), float(tt[1])
    ms_step = ms / a.steps
    value = B * world / (ms_step / 1000.0)

    # ---------------- e2e: host buffers through the pipelined public API ----
    e2e = None
    if a.e2e_steps > 0:
        # pinned host buffers for H and W: bound them to ~1/3 of host RAM across
        # the ranks of this node (a rate metric: a smaller sample is still valid)
        Be = H.shape[0]
        try:
            import psutil
            cap = int(psutil.virtual_memory().total / 3 / max(world, 1) / (2 * M * K * csz))
            Be = min(Be, max(256, cap))
        except Exception:  # noqa: BLE001
            pass
        pipe = BT.HostPipeline(M, K, dtype=dt, chunk=min(a.e2e_chunk, Be), device=dev)
        Hh = torch.empty(Be, M, K, dtype=dt, pin_memory=True)
        Hh.copy_(H[:Be])
        Wh = torch.empty_like(Hh, pin_memory=True)
        Sh = torch.empty(B, dtype=torch.float64, pin_memory=True)
        Sth = torch.empty(B, dtype=torch.int32, pin_memory=True)
        pipe.run(Hh, Wh, Sh, Sth, alpha, power, a.method, T)   # warm-up
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.e2e_steps):
            pipe.run(Hh, Wh, Sh, Sth, alpha, power, a.method, T)
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / a.e2e_steps
        if world > 1:
            tt = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt[0])
        L.raise_status(Sth.numpy(), "bench e2e")
        e2e = {"value": Be * world / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": Be * M * K * csz,
               "d2h_bytes_per_step": Be * M * K * csz + Be * (8 + 4),
               "ms_per_step": ems, "realizations_per_rank": Be,
               "path": f"HostPipeline (3 streams, {min(a.e2e_chunk, Be)}-realization chunks)"}
        # the e2e bound: pinned host<->device copies in both directions at once
        nb = min(Be, 1024)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        hd, dd = Hh[:nb], H[:nb]
        wd = torch.empty_like(dd)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        c0.record()
        for _ in range(3):
            with torch.cuda.stream(s1):
                wd.copy_(hd, non_blocking=True)
            with torch.cuda.stream(s2):
                Wh[:nb].copy_(dd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        c1.record()
        torch.cuda.synchronize()
        bw = 3 * nb * M * K * csz / (c0.elapsed_time(c1) / 1000.0)
        bound = bw / (M * K * csz) * world
        e2e["roofline"] = {"bound": "pcie", "achieved_gbs_per_direction": e2e["value"] * M * K * csz / world / 1e9,
                           "peak_gbs_per_direction": bw / 1e9, "peak_source": "pinned copies, both directions at once",
                           "frac": e2e["value"] / bound}
        del Hh, Wh, wd

    # ---------------- roofline of the fused precoder call -------------------
    hbm, bf16, peak_src = load_peaks()
    bytes_per = 2 * M * K * csz
    flops_per = flops_per_precoder(M, K, T, a.method)
    t_bytes = B * bytes_per / (hbm * 1e9)
    # tensor peak for the arithmetic actually used (3 fp16 MMAs per real product)
    tc_peak = bf16 / 3.0 if tc else None
    t_flop = B * flops_per / (tc_peak * 1e12) if tc_peak else 0.0
    bound = "tensor" if t_flop > t_bytes else "hbm"
    kern_s = kern_ms / 1000.0
    if bound == "hbm":
        achieved, peak, unit = B * bytes_per / kern_s / 1e9, hbm, "GB/s"
    else:
        achieved, peak, unit = B * flops_per / kern_s / 1e12, tc_peak, "TFLOP/s"
    # DRAM bytes per launch from the committed ncu --set full capture
    # (bytes per precoder there x this launch's realizations), or null
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            rec = json.load(f).get(f"{a.config}:{a.method}")
        if rec and tc:
            traffic = rec["dram_bytes_per_precoder"] * B
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": traffic,
            "peak_source": f"{peak_src} (MEASURED_PEAKS.json)" if peak_src == "measured" else peak_src,
            "kernel": ("xl_rzf precoder call" + (" (tcgen05)" if tc else " (general path)")
                       + (f", {B // sub} calls of {sub} per step" if sub < B else "")),
            "kernel_ms": kern_ms, "bytes_per_precoder": bytes_per,
            "algorithmic_bytes_per_launch": B * bytes_per,
            "traffic_source": "profiles/traffic.json" if traffic is not None else None,
            "flops_per_precoder": flops_per}
    # SURVEY.md section 8(d)'s convention, for comparison: c64 priced as
    # 3xTF32 (TF32 ~ BF16 / 2, so BF16 / 6), which makes cfg3 tensor-bound;
    # the 3xFP16 split used here runs at the FP16 (= BF16) rate, hence the
    # primary "roofline" above is the HBM bound.
    if tc:
        p3 = bf16 / 6.0
        t_roof = max(flops_per / (p3 * 1e12), bytes_per / (hbm * 1e9))
        roof["survey_convention"] = {
            "bound": "tensor" if flops_per / (p3 * 1e12) > bytes_per / (hbm * 1e9) else "hbm",
            "tensor_peak_tflops": p3, "roofline_precoders_per_s": 1.0 / t_roof,
            "frac": (B / kern_s) * t_roof}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a.config, a.method, a.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong" if gen_in_step else "weak", "vs_baseline": None,
                "dtype": "c64" if dt == torch.complex64 else "c128", "data": "synthetic",
                "config": {"workload": f"{a.config}: M={M}, K={K}, T={T}, {a.method}, "
                                       f"{B} realizations per GPU"
                                       + (f", generated on device in chunks of {sub} inside the step"
                                          if gen_in_step else
                                          (f", precoded in sub-batches of {sub}" if sub < B else "")),
                           "sub_batch": sub, "channel_generation_timed": gen_in_step,
                           "M": M, "K": K, "T": T, "batch_per_gpu": B,
                           "global_batch": B * world, "method": a.method,
                           "parallelism": f"realization-sharded x{world}",
                           "l2": f"inputs {B * M * K * csz / 2**30:.1f} GiB per GPU >> 126 MB L2"},
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
                "gpu_launches": launches, "clocks": clk.summary(),
                "ergodic_se": {"mean": float(se_mean[0]), "sem": float(se_mean[1]),
                               "realizations": B * world},
                "tensor_core_path": tc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
