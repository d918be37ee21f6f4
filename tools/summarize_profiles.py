#!/usr/bin/env python3
"""Summarise the ncu outputs of tools/prof_cmd.sh into profiles/ (committed evidence).

    python tools/summarize_profiles.py --round r01 [--launches gpurun_out/launches_bench.csv]
                                        [--full gpurun_out/prof_u2_100k.ncu-rep]

Writes:
  profiles/<round>_launches_summary.txt  per-kernel share of the launch list (ncu
                                          gpu__time_duration.sum, serialised, cold cache)
  profiles/<round>_launches.csv.gz       the raw launch list
  profiles/<round>_u2_full_summary.txt   key metrics of the --set full capture of one
                                          bulk trailing-update (U2) launch
  profiles/trailing_dram_bytes.json       dram read+write bytes per U2 launch (bench.py
                                          roofline.traffic) with the launch's algorithmic flops
"""
import argparse
import collections
import csv
import gzip
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def kernel_class(name: str) -> str:
    if "SyrkMap" in name:
        return "trail_update_kernel<SyrkMap> (trailing update U1/U2)"
    if "DenseMap" in name:
        return "panel_gemm_kernel / gemm_nt_dmma<DenseMap> (panel update / TRSM)"
    return name.split("(")[0].replace("exageo::<unnamed>::", "").replace("void ", "")[:60]


def summarize_launches(path: str, rnd: str):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        k = kernel_class(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    out = os.path.join(PROF, f"{rnd}_launches_summary.txt")
    with open(out, "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold cache)\n")
        f.write(f"# source: {os.path.basename(path)}; {sum(v[0] for v in agg.values())} launches profiled\n")
        f.write(f"{'launches':>9} {'total ms':>12} {'share':>7} {'avg us':>12}  kernel\n")
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{v[0]:9d} {v[1] / 1e3:12.2f} {100 * v[1] / tot:6.1f}% {v[1] / v[0]:12.1f}  {k}\n")
    with open(path, "rb") as fi, gzip.open(os.path.join(PROF, f"{rnd}_launches.csv.gz"), "wb") as fo:
        shutil.copyfileobj(fi, fo)
    print(open(out).read())


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def summarize_full(path: str, rnd: str, n: int, nb: int):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    got = {}
    for h, u, v in zip(hdr, units, vals):
        if h in METRICS:
            got[h] = (v, u)
    stalls = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st = sum(s for s, _ in stalls) or 1.0
    unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd = float(got["dram__bytes_read.sum"][0].replace(",", "")) * unit_scale.get(got["dram__bytes_read.sum"][1], 1)
    wr = float(got["dram__bytes_write.sum"][0].replace(",", "")) * unit_scale.get(got["dram__bytes_write.sum"][1], 1)
    tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}
    dur = float(got["gpu__time_duration.sum"][0].replace(",", "")) * tscale.get(got["gpu__time_duration.sum"][1], 1e-9)
    # the captured launch is U2(0) of an n x n problem: panels 2..T-1 updated by panel 0
    m = n - 2 * nb
    flops = 2.0 * nb * (m * (m + 1) / 2 + m)
    out = os.path.join(PROF, f"{rnd}_u2_full_summary.txt")
    with open(out, "w") as f:
        f.write(f"# ncu --set full --clock-control none, kernel trail_update_kernel<SyrkMap> U2(0) at n={n}, nb={nb}\n")
        for h in METRICS:
            if h in got:
                f.write(f"{h:80s} {got[h][0]:>18s} {got[h][1]}\n")
        f.write(f"\nalgorithmic flops of this launch: {flops:.4e}  ->  {flops / dur / 1e12:.2f} TFLOP/s under ncu "
                f"(serialised; bench.py reports the live figure)\n")
        f.write(f"dram traffic: read {rd / 1e9:.2f} GB + write {wr / 1e9:.2f} GB = {(rd + wr) / 1e9:.2f} GB; "
                f"algorithmic C read+write {2 * 8 * (m * (m + 1) / 2) / 1e9:.2f} GB\n")
        f.write("\nwarp stall samples (share):\n")
        for s, name in sorted(stalls, reverse=True)[:10]:
            f.write(f"  {name:30s} {100 * s / st:5.1f}%\n")
    json.dump({"dram_bytes_per_launch": rd + wr, "launch": f"U2(0) at n={n}, nb={nb}", "flops_per_launch": flops,
               "source": os.path.basename(out)}, open(os.path.join(PROF, "trailing_dram_bytes.json"), "w"), indent=1)
    print(open(out).read())


AUX_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
               "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
               "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
               "launch__registers_per_thread", "smsp__inst_executed.sum"]


def summarize_aux(paths, rnd: str):
    """Key metrics of --set full captures of the secondary kernels (generation, POTRF, ...)."""
    out = os.path.join(PROF, f"{rnd}_aux_kernels_summary.txt")
    with open(out, "w") as f:
        f.write("# ncu --set full --clock-control none captures of the secondary kernels (tools/prof_aux.sh)\n")
        for label, path in paths:
            raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rows = list(csv.reader(raw.splitlines()))
            if len(rows) < 3:
                continue
            hdr, units, vals = rows[0], rows[1], rows[2]
            got = {h: (v, u) for h, u, v in zip(hdr, units, vals) if h in AUX_METRICS}
            stalls = []
            for h, v in zip(hdr, vals):
                if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                    try:
                        stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            st = sum(x for x, _ in stalls) or 1.0
            f.write(f"\n== {label}  ({os.path.basename(path)})\n")
            for h in AUX_METRICS:
                if h in got:
                    f.write(f"  {h:72s} {got[h][0]:>16s} {got[h][1]}\n")
            f.write("  warp stall samples: " + ", ".join(f"{name} {100 * x / st:.0f}%"
                                                        for x, name in sorted(stalls, reverse=True)[:5]) + "\n")
    print(open(out).read())


def summarize_mid(items, rnd: str):
    """U2(0) captures at mid n (tools/r02_mid_profiles.sh): n:nb:path triples -> one table."""
    out = os.path.join(PROF, f"{rnd}_u2_mid_summary.txt")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
    unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}
    with open(out, "w") as f:
        f.write("# ncu --set full --clock-control none, trail_update_kernel<SyrkMap> U2(0) (panel 0 updating panels\n"
                "# 2..T-1) at mid n; algorithmic flops 2 nb (m(m+1)/2 + m), algorithmic C bytes 16 m(m+1)/2,\n"
                "# m = n - 2 nb. DRAM bytes per algorithmic flop fall with K = nb (the delayed-update lever).\n")
        f.write(f"{'n':>6s} {'nb':>5s} {'grid':>7s} {'time ms':>9s} {'TF/s':>6s} {'DMMA pipe':>9s} "
                f"{'DRAM GB':>8s} {'C alg GB':>8s} {'B/flop':>7s}\n")
        for n, nb, path in items:
            n, nb = int(n), int(nb)
            raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                                 text=True).stdout
            rows = list(csv.reader(raw.splitlines()))
            got = {h: (v.replace(",", ""), u) for h, u, v in zip(rows[0], rows[1], rows[2]) if h in keys}
            dur = float(got[keys[0]][0]) * tscale.get(got[keys[0]][1], 1e-9)
            dram = sum(float(got[k][0]) * unit_scale.get(got[k][1], 1) for k in keys[1:3])
            m = n - 2 * nb
            flops = 2.0 * nb * (m * (m + 1) / 2 + m)
            f.write(f"{n:6d} {nb:5d} {got[keys[4]][0]:>7s} {dur * 1e3:9.3f} {flops / dur / 1e12:6.2f} "
                    f"{float(got[keys[3]][0]):8.1f}% {dram / 1e9:8.3f} {16 * m * (m + 1) / 2 / 1e9:8.3f} "
                    f"{dram / flops:7.4f}\n")
    print(open(out).read())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--aux", nargs="*", default=None, help="label::path.ncu-rep pairs for summarize_aux")
    ap.add_argument("--mid", nargs="*", default=None, help="n:nb:path.ncu-rep triples for summarize_mid")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches_bench.csv"))
    ap.add_argument("--full", default=os.path.join(ROOT, "gpurun_out", "prof_u2_100k.ncu-rep"))
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--nb", type=int, default=512)
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.mid:
        summarize_mid([tuple(x.split(":", 2)) for x in a.mid], a.round)
        return
    if a.aux:
        summarize_aux([tuple(x.split("::", 1)) for x in a.aux], a.round)
        return
    if os.path.exists(a.launches):
        summarize_launches(a.launches, a.round)
    if os.path.exists(a.full):
        summarize_full(a.full, a.round, a.n, a.nb)


if __name__ == "__main__":
    main()
