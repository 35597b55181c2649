"""Benchmark: Jac-PCG RZF precoders/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
                    [--scaling strong|weak] [--impl ours|reference]

A step = one pass of the hot path over one batch resident in HBM: the
batched precoder (Gram -> Jac-PCG T iterations -> beta, W -> SINR/SE) for the
rank's realizations, plus the ergodic-SE partials (and their NCCL all-gather
when N > 1).  cfg4 generates its channels on device in chunks inside the step
(generation of chunk n + 1 overlaps precoding of chunk n on a second stream);
cfg2 runs the whole paired grid (T in {2..5} x {jacpcg, cg, direct} x 7 SNR
points on one batch) per step.

Scaling (distributed.rank_batch): "strong" (default, as the BASELINE configs
state them: the config's batch is split over the N GPUs) or "weak" (every
GPU owns the config's batch).

Prints ONE JSON line on rank 0 (contract in the task statement):
value = precoders/s of the whole job (device-timed, CUDA events, max over
ranks), e2e = the same metric through the host-buffer API (pinned H in, W and
SE out, copies inside the timed region), roofline of the precoder call
(algorithmic bytes and flops vs the measured peaks of the arithmetic the path
runs), cpu_baseline = the CPU oracle port on this host's cores (rank 0,
N = 1) plus a parity sample of the timed batch checked against it.
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


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--batch", type=int, default=None, help="override the config's batch")
    ap.add_argument("--method", default="jacpcg")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=256,
                    help="realizations per HostPipeline chunk (fill/drain ~ 1/number of chunks)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--parity-sample", type=int, default=None,
                    help="realizations of the timed batch checked against the oracle (rank 0, N = 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args(argv)


# --------------------------------------------------------------- helpers ----

def load_peaks():
    """HBM GB/s and dense tensor TFLOP/s of the arithmetic each path runs:
    MEASURED_PEAKS.json (driver: copy bandwidth, bf16 = fp16 rate) and
    profiles/r02_peaks_tf32_fp64.json (measured on the box, tools/measure_peaks.py:
    TF32, FP64 and FP32-SIMT GEMM rates)."""
    out = {"hbm": 6650.0, "fp16": 1590.0, "src": "fallback (B200_PROFILING.md)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        out.update(hbm=d.get("hbm_gbs", 6650.0), fp16=d.get("bf16_tflops", 1590.0),
                   src="measured (MEASURED_PEAKS.json)")
    q = os.path.join(ROOT, "profiles", "r02_peaks_tf32_fp64.json")
    out.update(tf32=None, fp64=None, fp32=None, mma_sync=None)
    r = os.path.join(ROOT, "profiles", "r02_peaks_mma_sync.json")
    if os.path.exists(r):
        with open(r) as f:
            out.update(mma_sync=json.load(f).get("mma_sync_fp16_tflops"))
    if os.path.exists(q):
        with open(q) as f:
            d = json.load(f)
        out.update(tf32=d.get("tf32_tflops"), fp64=d.get("fp64_tflops"), fp32=d.get("fp32_simt_tflops"))
    return out


def roofline(M, K, T, method, dtype_bytes, B, kern_ms, path, peaks, traffic=None):
    """Slower of tensor FLOPs at the peak of the arithmetic actually run and
    H/W bytes at HBM bandwidth (north_star); frac of the binding bound."""
    from paper_2305_13925_b200.flops import precoder_bytes, precoder_flops
    bytes_per = precoder_bytes(M, K, dtype_bytes)
    flops_per = precoder_flops(M, K, T, method)
    # tensor peak for the arithmetic the path executes
    if path == "tc3xfp16":      # 3 fp16 MMAs per real product on tcgen05
        tpeak, tname = peaks["fp16"] / 3.0, "fp16 tensor / 3 (3xFP16 split on tcgen05)"
    elif path == "mma3xfp16":   # 3 fp16 mma.sync per real product (warp-level tensor cores)
        tpeak = (peaks.get("mma_sync") or 550.0) / 3.0
        tname = "fp16 mma.sync / 3 (3xFP16 split, measured legacy-MMA rate)"
    elif path == "fp64":
        tpeak, tname = peaks["fp64"] or 35.0, "FP64 (DMMA / DFMA GEMM rate, measured)"
    else:                       # fp32 SIMT kernels
        tpeak, tname = peaks["fp32"] or 64.0, "FP32 SIMT (measured SGEMM rate)"
    t_bytes = B * bytes_per / (peaks["hbm"] * 1e9)
    t_flop = B * flops_per / (tpeak * 1e12)
    kern_s = kern_ms / 1000.0
    hbm_ach = B * bytes_per / kern_s / 1e9
    fl_ach = B * flops_per / kern_s / 1e12
    if t_flop > t_bytes:
        bound, achieved, peak, unit = "tensor", fl_ach, tpeak, "TFLOP/s"
    else:
        bound, achieved, peak, unit = "hbm", hbm_ach, peaks["hbm"], "GB/s"
    r = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
         "frac": achieved / peak, "traffic": traffic,
         "peak_source": peaks["src"], "tensor_peak": tname, "tensor_peak_tflops": tpeak,
         "frac_hbm": hbm_ach / peaks["hbm"], "frac_tensor": fl_ach / tpeak,
         "roofline_precoders_per_s": 1.0 / max(t_flop / B, t_bytes / B),
         "kernel_ms": kern_ms, "bytes_per_precoder": bytes_per,
         "algorithmic_bytes_per_launch": B * bytes_per, "flops_per_precoder": flops_per}
    return r


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
        self.samples, self.power, self.reasons, self.max_mhz = [], [], set(), None
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
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
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
                "power_w_median": statistics.median(self.power) if self.power else None,
                "power_limit_w": self.limit_w, "samples": len(self.samples)}


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
    from paper_2305_13925_b200.configs import CONFIGS
    return {"value": n / el, "unit": UNIT, "cores": cores, "kind": "port",
            "single_core_value": n1 / el1, "cpu_model": model,
            "sample": f"{n} {cfg_name} precoders ({method}, T={CONFIGS[cfg_name].T}) + SINR/SE, "
                      f"complex128 oracle, {cores} processes x 1 BLAS thread, {el:.1f} s"}


def parity_sample(H, out, idx, xi, power, method, T, sigma2=1.0):
    """Checker of the timed batch (cpu_baseline leg): the oracle on the
    realizations ``idx`` of the batch the timed steps precoded, compared with
    the device's W and sum-SE (relative Frobenius / relative)."""
    import numpy as np
    from oracle import xlmimo_oracle as O
    Hn = H[idx].cpu().numpy().astype(np.complex128)
    W = out.W[idx].cpu().numpy().astype(np.complex128)
    se = out.sum_se[idx].cpu().numpy()
    werr, serr = [], []
    for i in range(len(idx)):
        G, _, _, s = O.precoder_and_se(Hn[i], xi, power, sigma2, method, T, "textbook")
        werr.append(float(np.linalg.norm(W[i] - G) / np.linalg.norm(G)))
        serr.append(abs(float(se[i]) - s) / abs(s))
    return {"realizations": len(idx), "max_w_rel_err": max(werr), "max_se_rel_err": max(serr),
            "median_w_rel_err": float(np.median(werr)),
            "checked": "oracle (complex128 numpy restatement of the reference) on the timed batch"}


# ------------------------------------------------------------------ reference arm --

def _ref_config(a, wl, world):
    from paper_2305_13925_b200.distributed import rank_batch
    B = a.batch or wl.B
    _, nb = rank_batch(a.scaling, B, world, 0)
    csz = 16 if "128" in str(wl.dtype) else 8
    return {"workload": f"{a.config}: M={wl.M}, K={wl.K}, T={wl.T}, {a.method}, "
                        f"{nb} realizations per GPU",
            "M": wl.M, "K": wl.K, "T": wl.T, "method": a.method, "variant": "textbook",
            "dtype": "c64" if "128" not in str(wl.dtype) else "c128",
            "global_batch": B if a.scaling == "strong" else B * world,
            "batch_per_gpu": nb, "scaling": a.scaling,
            "parallelism": f"realization-sharded x{world}",
            # properties of the workload, stated as on our arm
            "channel_generation_timed": wl.chunk is not None,
            "l2": (f"inputs {nb * wl.M * wl.K * csz / 2**30:.2f} GiB per GPU >> 126 MB L2"
                   if nb * wl.M * wl.K * csz > 2**28 else "inputs below 256 MiB")}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
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
    cfg = _ref_config(a, wl, world)
    cb["sample"] = (f"reference algorithm (CPU port, complex128), per-step sample of {secs:.0f} s; "
                    + str(cb.get("sample", "")))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1000.0 * secs, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": cfg, "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm ----

def path_of(X, dt, method, M, K):
    import torch
    tc = X.tensor_core_path(dt, method, M, K)
    if tc in ("tcgen05", "tcgen05+mma.sync"):  # the latter: Gram / W (most flops) on tcgen05
        return "tc3xfp16"
    if tc == "mma.sync":
        return "mma3xfp16"
    return "fp64" if dt == torch.complex128 else "fp32"


def main(argv=None):
    a = parse(argv)
    if a.impl == "reference":
        run_reference(a)
        return
    if a.config == "cfg2":
        return run_grid(a)

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
    from paper_2305_13925_b200.distributed import DeviceTimer, ergodic_se, max_over_ranks, rank_batch

    wl = X.CONFIGS[a.config]
    M, K, T = wl.M, wl.K, wl.T
    dt = wl.dtype
    csz = 8 if dt == torch.complex64 else 16
    total = a.batch or wl.B
    first, B = rank_batch(a.scaling, total, world, rank)
    # cfg4 (configs[3]): generated on device in chunks of 2048 per GPU inside the
    # step (65536 do not fit HBM at once: 256 GiB); other configs: the rank's
    # batch is resident in HBM, precoded in one call or in sub-batches (below)
    gen_in_step = wl.chunk is not None
    if gen_in_step:
        sub = min(wl.chunk, B)
    else:
        # one call per step while H, W and the K x K state fit comfortably in
        # HBM (cfg5 c64: 32 GiB each of H and W); otherwise 2048-realization calls
        sub = B if B * M * K * csz <= 32 * 2**30 and dt == torch.complex64 else (
            B if B * M * K * csz <= 16 * 2**30 else 2048)
    assert B % sub == 0, "batch must be a multiple of the sub-batch"
    alpha, power = wl.alpha(), wl.power()
    lib = L.lib()
    path = path_of(X, dt, a.method, M, K)
    nbuf = 2 if gen_in_step else 1
    if gen_in_step:
        Hbuf = [torch.empty(sub, M, K, dtype=dt, device=dev) for _ in range(nbuf)]
        H = Hbuf[0]
        s_gen = torch.cuda.Stream(dev)
        ev_gen = [torch.cuda.Event() for _ in range(nbuf)]
        ev_used = [torch.cuda.Event() for _ in range(nbuf)]
    else:
        H = X.generate_channels(wl.model, seed=0, first=first, B=B, dtype=dt, device=dev)
    outs = [BT.alloc_outputs(H[:sub], want_gamma=True) for _ in range(nbuf)]
    se_all = torch.empty(B, dtype=torch.float64, device=dev)
    st_all = torch.empty(B, dtype=torch.int32, device=dev)
    comp = torch.cuda.current_stream(dev)

    def step(record=None):
        nch = B // sub
        if gen_in_step:   # chunk 0's channels; later chunks are generated one ahead
            with torch.cuda.stream(s_gen):
                s_gen.wait_event(ev_used[0])
                X.generate_channels(wl.model, seed=0, first=first, B=sub, dtype=dt, device=dev,
                                    out=Hbuf[0], check=False)
                ev_gen[0].record(s_gen)
        for ci in range(nch):
            c0 = ci * sub
            j = ci % nbuf
            if gen_in_step:
                if ci + 1 < nch:   # generate chunk ci + 1 on the side stream meanwhile
                    jn = (ci + 1) % nbuf
                    with torch.cuda.stream(s_gen):
                        s_gen.wait_event(ev_used[jn])
                        X.generate_channels(wl.model, seed=0, first=first + c0 + sub, B=sub, dtype=dt,
                                            device=dev, out=Hbuf[jn], check=False)
                        ev_gen[jn].record(s_gen)
                comp.wait_event(ev_gen[j])
                Hc = Hbuf[j]
            else:
                Hc = H[c0:c0 + sub]
            if record is not None:
                record[ci][0].record()
            BT.rzf_batched(Hc, alpha, power, method=a.method, T=T, variant="textbook", sigma2=1.0,
                           out=outs[j], check=False)
            if record is not None:
                record[ci][1].record()
            if gen_in_step:
                ev_used[j].record(comp)
            if sub < B:
                se_all[c0:c0 + sub].copy_(outs[j].sum_se)
                st_all[c0:c0 + sub].copy_(outs[j].status)
        return ergodic_se(outs[0].sum_se if sub == B else se_all, chunk=2048,
                          group=None if world > 1 else False)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    L.raise_status((outs[0].status if sub == B else st_all).cpu().numpy(), "bench warm-up")

    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(B // sub)] for _ in range(a.steps)]
    # small single-call batches (cfg1: 100 realizations) are bound by host launch
    # overhead: the step (precoder call + ergodic-SE partials) is captured once
    # into a CUDA graph and replayed (streams and graphs, no tracing compiler)
    graphed = (not gen_in_step) and sub == B and B <= 4096 and world == 1
    if graphed:
        n_eager = lib.xl_launch_count()
        step()
        torch.cuda.synchronize()
        per_step_launches = int(lib.xl_launch_count() - n_eager)
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(torch.cuda.current_stream(dev))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            g_out = step()
        torch.cuda.synchronize()
    n0 = lib.xl_launch_count()
    with ClockSampler(local) as clk:
        with DeviceTimer(dev) as timer:
            for i in range(a.steps):
                if graphed:
                    ev[i][0][0].record()
                    graph.replay()
                    ev[i][0][1].record()
                    se_mean = g_out
                else:
                    se_mean = step(ev[i])
    launches = per_step_launches * a.steps if graphed else int(lib.xl_launch_count() - n0)
    # the precoder calls of one step (without the in-step channel generation)
    kern_ms = statistics.mean(sum(e0.elapsed_time(e1) for e0, e1 in evs) for evs in ev)
    kern_ms = max_over_ranks([kern_ms], dev)[0]
    ms_step = timer.ms / a.steps
    value = total / (ms_step / 1000.0) if a.scaling == "strong" else B * world / (ms_step / 1000.0)
    L.raise_status((outs[0].status if sub == B else st_all).cpu().numpy(), "bench timed steps")

    # ---------------- e2e: host buffers through the pipelined public API ----
    e2e = None
    if a.e2e_steps > 0:
        # pinned host buffers for H and W: bound them to ~1/3 of host RAM across
        # the ranks of this node (a rate metric: a smaller sample is still valid)
        Be = min(B, H.shape[0])
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
        Sh = torch.empty(Be, dtype=torch.float64, pin_memory=True)
        Sth = torch.empty(Be, dtype=torch.int32, pin_memory=True)
        pipe.run(Hh, Wh, Sh, Sth, alpha, power, a.method, T)   # warm-up
        with DeviceTimer(dev) as et:
            for _ in range(a.e2e_steps):
                pipe.run(Hh, Wh, Sh, Sth, alpha, power, a.method, T)
        ems = et.ms / a.e2e_steps
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

    # ---------------- roofline of the precoder call --------------------------
    peaks = load_peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            rec = json.load(f).get(f"{a.config}:{a.method}")
        if rec:
            traffic = rec["dram_bytes_per_precoder"] * B
    roof = roofline(M, K, T, a.method, csz, B, kern_ms, path, peaks, traffic)
    roof["kernel"] = ("xl_rzf precoder call" + {"tc3xfp16": " (tcgen05)", "fp64": " (c128 path)",
                                                  "fp32": " (SIMT path)"}[path]
                      + (f", {B // sub} calls of {sub} per step" if sub < B else ""))
    if traffic is not None:
        roof["traffic_source"] = "profiles/traffic.json"
    if a.config == "cfg3" and path == "tc3xfp16":
        # measured energy model under the 1000 W board cap (profiles/r01_power.md)
        roof["power_roofline"] = {"precoders_per_s": 5.4e6, "frac": value / world / 5.4e6,
                                  "source": "profiles/r01_power.md (unavoidable data movement at 1000 W)"}

    cpu = parity = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a.config, a.method, a.cpu_seconds)
        # the checker leg: oracle on a sample of the last sub-batch the timed steps precoded
        n_par = a.parity_sample if a.parity_sample is not None else (64 if M * K <= 65536 else 16)
        last = (B // sub - 1) % nbuf
        Hlast = Hbuf[last] if gen_in_step else H[B - sub:B]
        idx = sorted(set(int(round(i * (sub - 1) / max(1, n_par - 1))) for i in range(n_par)))
        parity = parity_sample(Hlast, outs[last], idx, alpha, power, a.method, T)
        cpu["parity_sample"] = parity

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
                "dtype": "c64" if dt == torch.complex64 else "c128", "data": "synthetic",
                "config": {"workload": f"{a.config}: M={M}, K={K}, T={T}, {a.method}, "
                                       f"{B} realizations per GPU"
                                       + (f", generated on device in chunks of {sub} inside the step "
                                          f"(generation of chunk n+1 overlaps precoding of chunk n)"
                                          if gen_in_step else
                                          (f", precoded in sub-batches of {sub}" if sub < B else "")),
                           "channel_generation_timed": gen_in_step,
                           "M": M, "K": K, "T": T, "method": a.method, "variant": "textbook",
                           "dtype": "c64" if dt == torch.complex64 else "c128",
                           "batch_per_gpu": B, "global_batch": total if a.scaling == "strong" else B * world,
                           "scaling": a.scaling,
                           "parallelism": f"realization-sharded x{world}",
                           "l2": f"inputs {B * M * K * csz / 2**30:.2f} GiB per GPU >> 126 MB L2"
                                 if B * M * K * csz > 2**28 else "inputs below 256 MiB"},
                "harness": {"sub_batch": sub, "cuda_graph": graphed},
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
                "gpu_launches": launches, "clocks": clk.summary(),
                "ergodic_se": {"mean": float(se_mean[0]), "sem": float(se_mean[1]),
                               "realizations": total if a.scaling == "strong" else B * world},
                "tensor_core_path": path == "tc3xfp16"}
        if parity is not None:
            line["parity_sample"] = parity
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------- cfg2: paired grid ----

def run_grid(a):
    """configs[1]: T in {2,3,4,5} x {jacpcg, cg, direct} x SNR -10..20 dB on one
    paired batch of 8192 realizations; a step = every grid point once."""
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
    from paper_2305_13925_b200 import trials as TR
    from paper_2305_13925_b200.distributed import DeviceTimer, max_over_ranks, rank_batch

    wl = X.CONFIGS["cfg2"]
    M, K = wl.M, wl.K
    total = a.batch or wl.B
    first, B = rank_batch(a.scaling, total, world, rank)
    H = X.generate_channels(wl.model, seed=0, first=first, B=B, dtype=wl.dtype, device=dev)
    pts = TR.grid_points(("jacpcg", "cg", "direct"), (2, 3, 4, 5), wl.snr_grid_db)
    lib = L.lib()
    for _ in range(a.warmup):
        TR.se_grid_batched(H, pts, check=True)
    torch.cuda.synchronize()
    # the step (63 launches over two streams) is captured once and replayed, so
    # no host-side delay between launches enters the timed region
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cap):
        TR.se_grid_batched(H, pts, check=False)   # side streams / workspaces exist before capture
        cap.synchronize()
        n_cap = lib.xl_launch_count()
        with torch.cuda.graph(graph, stream=cap):
            g_graph = TR.se_grid_batched(H, pts, check=False)
        launches_per_step = int(lib.xl_launch_count() - n_cap)
    torch.cuda.current_stream(dev).wait_stream(cap)
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with DeviceTimer(dev) as timer:
            for _ in range(a.steps):
                graph.replay()
    launches = launches_per_step * a.steps
    for p in pts:
        L.raise_status(g_graph.status[p].cpu().numpy(), f"bench grid {p}")
    # per-point device times: separate direct (non-graph) passes, outside the timed region
    # (a ~2 ms device sleep first keeps the GPU busy while the host enqueues, so
    # the first point's events do not time the host's launch latency)
    # (the previous pass's outputs are released first so its scratch W is reused, not re-allocated)
    per_point = {p: [] for p in pts}
    g = None
    for _ in range(4):
        g = None
        torch.cuda._sleep(4_000_000)
        g = TR.se_grid_batched(H, pts, timed=True, check=False, lanes=1)
        if _ == 0:
            continue  # warm pass
        for p in pts:
            per_point[p].append(g.ms[p])
    grids = [g_graph]
    ms_step = timer.ms / a.steps
    n_prec = len(pts) * (total if a.scaling == "strong" else B * world)
    value = n_prec / (ms_step / 1000.0)
    peaks = load_peaks()
    rows = []
    for p in pts:
        ms = max_over_ranks([statistics.mean(per_point[p])], dev)[0]
        path = path_of(X, wl.dtype, p.method, M, K)
        r = roofline(M, K, max(p.T, 1), p.method, 8, B, ms, path, peaks)
        rows.append({"method": p.method, "T": p.T, "snr_db": p.snr_db, "ms": ms,
                     "precoders_per_s": B * world / (ms / 1000.0), "path": path,
                     "roofline_bound": r["bound"], "roofline_frac": r["frac"]})
    erg = grids[-1].ergodic()
    # the grid's representative point (jacpcg T = 4, 10 dB) carries the roofline object
    rep = next(p for p in pts if p.method == "jacpcg" and p.T == 4 and p.snr_db == 10.0)
    roof = roofline(M, K, 4, "jacpcg", 8, B, max_over_ranks([statistics.mean(per_point[rep])], dev)[0],
                    path_of(X, wl.dtype, "jacpcg", M, K), peaks)
    roof["kernel"] = "xl_rzf fused call at jacpcg T=4, 10 dB (tcgen05); per-point fractions under grid"

    # e2e through the public API: H from pinned host once per step (all points are
    # paired on it), every point's sum-SE back to pinned host.  The batch moves in
    # two halves on a copy stream: the grid runs on half 0 while half 1 crosses PCIe.
    Hh = torch.empty(B, M, K, dtype=wl.dtype, pin_memory=True)
    Hh.copy_(H)
    Sh = torch.empty(len(pts), B, dtype=torch.float64, pin_memory=True)
    Hd = torch.empty_like(H)
    s_copy = torch.cuda.Stream(dev)
    halves = [(0, B // 2), (B // 2, B)] if B >= 2 else [(0, B)]
    ev_in = [torch.cuda.Event() for _ in halves]

    def e2e_step():
        cur = torch.cuda.current_stream(dev)
        s_copy.wait_stream(cur)  # the previous step's grid has finished reading Hd
        with torch.cuda.stream(s_copy):
            for (lo, hi), ev in zip(halves, ev_in):
                Hd[lo:hi].copy_(Hh[lo:hi], non_blocking=True)
                ev.record(s_copy)
        for (lo, hi), ev in zip(halves, ev_in):
            cur.wait_event(ev)
            g = TR.se_grid_batched(Hd[lo:hi], pts, check=False)
            for i, p in enumerate(pts):
                Sh[i, lo:hi].copy_(g.sum_se[p], non_blocking=True)

    e2e_step()
    with DeviceTimer(dev) as et:
        for _ in range(max(1, a.e2e_steps)):
            e2e_step()
    ems = et.ms / max(1, a.e2e_steps)
    e2e = {"value": n_prec / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": B * M * K * 8,
           "d2h_bytes_per_step": len(pts) * B * 8, "ms_per_step": ems,
           "path": "H pinned host -> device once (two halves on a copy stream, the second overlapping "
                   "the grid on the first), trials.se_grid_batched (63 paired points), sum-SE back"}

    cpu = parity = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline("cfg2", "jacpcg", a.cpu_seconds)
        g = TR.se_grid_batched(H, [rep], keep_W=True, check=True)

        class _O:
            W = g.W[rep]
            sum_se = g.sum_se[rep]
        n_par = a.parity_sample or 64
        idx = sorted(set(int(round(i * (B - 1) / max(1, n_par - 1))) for i in range(n_par)))
        parity = parity_sample(H, _O, idx, TR.default_xi(K, 10.0), 10.0, "jacpcg", 4)
        cpu["parity_sample"] = parity
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": a.scaling, "vs_baseline": None, "dtype": "c64", "data": "synthetic",
                "config": {"workload": f"cfg2: M={M}, K={K}, paired grid T in {{2,3,4,5}} x "
                                       f"{{jacpcg, cg, direct}} x SNR {list(wl.snr_grid_db)} dB "
                                       f"({len(pts)} points) on {B} realizations per GPU",
                           "M": M, "K": K, "T": "2-5", "method": "grid", "dtype": "c64",
                           "batch_per_gpu": B, "global_batch": total if a.scaling == "strong" else B * world,
                           "points": len(pts), "scaling": a.scaling,
                           "cuda_graph": True, "streams": 2,
                           "parallelism": f"realization-sharded x{world}",
                           "l2": f"inputs {B * M * K * 8 / 2**20:.0f} MiB per GPU (reused by all points)"},
                "grid": rows,
                "ergodic_se": {f"{p.method}:T{p.T}:{p.snr_db:g}dB": {"mean": m, "sem": s}
                               for p, (m, s) in erg.items()},
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches,
                "clocks": clk.summary(), "tensor_core_path": True}
        if parity is not None:
            line["parity_sample"] = parity
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
