"""Write profiles/<round>_launches.md, profiles/<round>_fused_full.md and
profiles/traffic.json from the gpurun_out/ artifacts of tools/profile_round.sh.

usage: python tools/summarize_profiles.py r01 [live_ms]
"""
import collections
import csv
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
LIVE = sys.argv[2] if len(sys.argv) > 2 else None
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches():
    rows = list(csv.reader(open(os.path.join(OUT, f"{R}_launches.csv"))))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))

    def us(d):
        v = float(d["Metric Value"].replace(",", ""))
        return v * {"ms": 1e3, "us": 1, "ns": 1e-3, "s": 1e6, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}.get(d["Metric Unit"], 1)

    L = [(d["Kernel Name"], us(d)) for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
    out = [f"# {R}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
           "Command: `python bench.py` (cfg3, B = 32768, 3 warm-up + 10 timed steps, e2e 1 + 3 pipeline runs),",
           "profiled with `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv` (tools/profile_round.sh).",
           f"Raw list: `{R}_launches.csv`. ncu serialises launches and runs them cold: compare SHARES, not absolutes.", "",
           "## All launches of the command", "", "| launches | total ms | share | kernel |", "|---:|---:|---:|---|"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in L:
        agg[k[:70]][0] += 1
        agg[k[:70]][1] += t
    tot = sum(v[1] for v in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {n} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | `{k}` |")
    steps = []
    for i, (k, t) in enumerate(L):
        if "fused_rzf" in k and t > 5000:
            j, extra = i + 1, 0.0
            while j < len(L) and "fused_rzf" not in L[j][0] and "chan_kernel" not in L[j][0] and j - i < 15:
                extra += L[j][1]
                j += 1
            steps.append((t, extra))
    ft = sum(a for a, _ in steps) / len(steps)
    et = sum(b for _, b in steps) / len(steps)
    out += ["", "## One bench step (B = 32768)", "",
            f"Fused precoder kernel: {ft / 1e3:.3f} ms per launch under ncu ({len(steps)} launches); the SE reduction after it: {et:.1f} us.",
            f"Share of the step spent in `fused_rzf_kernel<64>`: **{100 * ft / (ft + et):.2f}%**."
            + (f" The live (non-profiled) bench measured {LIVE} ms per launch." if LIVE else "")]
    open(os.path.join(PROF, f"{R}_launches.md"), "w").write("\n".join(out) + "\n")
    subprocess.run(["cp", os.path.join(OUT, f"{R}_launches.csv"), os.path.join(PROF, f"{R}_launches.csv")], check=True)


def full():
    rep = os.path.join(OUT, f"{R}_fused.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    with open("/tmp/_src.csv", "w") as f:
        f.write(src)
    stalls = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), "/tmp/_src.csv", "16"],
                            capture_output=True, text=True).stdout
    B = 4096
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}

    def g(n):
        i = h.index(n)
        return float(v[i].replace(",", "")) * scale.get(u[i], 1)

    rdb, wrb = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    per, alg = (rdb + wrb) / B, 2 * 1024 * 64 * 8
    L = [f"# {R}: `ncu --set full` capture of the fused precoder kernel", "",
         "Command (tools/profile_round.sh): `ncu --set full --clock-control none --import-source on -k regex:fused_rzf "
         "-s 3 -c 1 python bench.py --batch 4096 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline`",
         "(cfg3: M = 1024, K = 64, T = 4, c64; 4096 realizations in one launch, 148 CTAs).",
         "Per-launch times under ncu are cold-cache and serialised; the bench number is the live one.", "",
         "| metric | value |", "|---|---|"]
    for n in ["launch__block_size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "launch__shared_mem_per_block_dynamic"]:
        if n in h:
            i = h.index(n)
            L.append(f"| `{n}` | {v[i]} {u[i]} |")
    L += ["", f"**DRAM traffic per precoder: {per / 1e6:.3f} MB** (read {rdb / B / 1e6:.3f} + write {wrb / B / 1e6:.3f}) "
          f"against the algorithmic 1.049 MB (read H once + write W: 2 x M x K x 8 B); ratio {per / alg:.2f}.",
          "The W pass re-reads H: its reuse distance is two ring passes (~1 MiB per SM, ~150 MB chip-wide), beyond L2",
          "(DESIGN.md section 6).", "", "## Where the warps stall (top source lines, `--page source`)", "", "```"]
    L += stalls.splitlines() + ["```", "",
          "Reading: conversion (LDS.128 of the raw fp32 tile -> packed fp16 hi/lo split -> core-matrix STS) and the W^T",
          "epilogue's streaming stores dominate the converter warps; the math warps' time spreads over the PCG phases;",
          "`sleep` samples at the final `__syncthreads` are the MMA-issuer / producer warps' idle lanes 1-31."]
    open(os.path.join(PROF, f"{R}_fused_full.md"), "w").write("\n".join(L) + "\n")
    json.dump({"cfg3:jacpcg": {"dram_bytes_per_precoder": per, "read_bytes_per_precoder": rdb / B,
                               "write_bytes_per_precoder": wrb / B,
                               "source": f"profiles/{R}_fused_full.md (ncu --set full, batch 4096)"}},
              open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    print("traffic per precoder", per, per / alg)


launches()
full()
