#!/usr/bin/env python3
"""bench.py -- exact Gaussian log-likelihood evaluations per second on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 100000] [--impl reference]

One "step" = one whole evaluation of the hot path (Alg. 2): Matern
generation + tiled Cholesky with fused forward solve + log-det/dot reduction,
at BASELINE.json's headline workload (n = 100k jittered-grid locations,
theta = (1, 0.1, 0.5), z = L(theta) e from a fixed seed; configs[2]).
Inputs (40.6 GB of tiles) are far larger than L2, so no flush is needed.

Prints ONE JSON line (rank 0). `value` = evaluations/s of the whole job with
inputs resident in HBM (exageo_loglik_dev); `e2e` = the same through the
host-pointer API exageo_loglik with pinned host buffers (H2D of x, y, z and
D2H of the result inside the timed region). `roofline` reports the dominant
kernel (the bulk DMMA trailing update) against the measured FP64 DMMA peak.
`--impl reference` times the CPU oracle (oracle/, the reference arm of this
tier) on a bounded sample and scales it to the same metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "loglik evals/sec at n=100k (1 GPU)"
UNIT = "evals/s"
THETA = (1.0, 0.1, 0.5)
SEED = 1


def fp64_peaks():
    """FP64 roofline denominators measured on this pool's B200 by tools/fp64_peak.sh and
    committed as profiles/fp64_peak.txt (MEASURED_PEAKS.json has no FP64 entry): the
    sustained DMMA.8x8x4 loop and cuBLAS DGEMM 8192^3 as the vendor yardstick."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.txt")
    dmma, dgemm, clocks = None, None, None
    for line in open(path):
        if line.startswith("DMMA sustained:"):
            dmma = float(line.split(":")[1].split()[0])
        elif line.startswith("cublas dgemm 8192^3:"):
            dgemm = float(line.split(":")[1].split()[0])
        elif line.startswith("clocks:"):
            clocks = line.strip()
    if dmma is None or dgemm is None:
        raise RuntimeError(f"{path}: DMMA / DGEMM lines missing (run tools/fp64_peak.sh on a B200)")
    return dmma, dgemm, f"measured: profiles/fp64_peak.txt (tools/fp64_peak.sh; {clocks})"


FP64_PEAK_TFLOPS, DGEMM_TFLOPS, FP64_PEAK_SOURCE = fp64_peaks()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clock / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                p = [v.strip() for v in line.split(",")]
                if len(p) >= 7:
                    try:
                        rows.append((float(p[0]), float(p[1]), float(p[2]), p[3:7]))
                    except ValueError:
                        pass
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [r for r in rows if r[2] > 300.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows), "samples": len(rows), "reasons": reasons}


# ----------------------------------------------------------------------------- oracle baseline
def oracle_sample(n_sample: int, n_target: int):
    """Time the CPU oracle on a bounded sample and scale to one evaluation at n_target.

    Generation (O(n^2) Matern/Bessel evaluations) and factorization+solve (O(n^3))
    are timed separately and scaled by (n_target/n_sample)^2 and ^3."""
    import numpy as np

    import oracle
    import synth_inputs as si

    x, y = oracle.gen_locations(n_sample, SEED)
    z = si.normals(n_sample, SEED)
    t0 = time.perf_counter()
    S = oracle.cov(x, y, x, y, THETA)
    t1 = time.perf_counter()
    L = oracle.cholesky(S)
    w = oracle.forward(L, z)
    _ = float(2 * np.log(np.diag(L)).sum() + w @ w)
    t2 = time.perf_counter()
    r = n_target / n_sample
    t_target = (t1 - t0) * r**2 + (t2 - t1) * r**3
    return {"t_gen": t1 - t0, "t_chol": t2 - t1, "t_total": t2 - t0, "t_target": t_target,
            "cores": oracle.num_threads()}


def oracle_measured() -> list:
    """Whole oracle evaluations actually run (not extrapolated): the committed goldens of
    tools/make_golden_large.py at n = 20k / 40k, with their seconds, threads and CPU model."""
    import glob

    out = []
    for f in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "loglik_n*.json"))):
        g = json.load(open(f))
        for c in g["cases"]:
            out.append({"n": g["n"], "theta": c["theta"], "seconds": c["oracle_seconds"],
                        "evals_per_s": 1.0 / c["oracle_seconds"], "threads": g["oracle_threads"],
                        "cpu_model": g["cpu_model"], "host": g.get("host"), "source": os.path.relpath(f, ROOT)})
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n_sample = args.ref_sample
    for _ in range(args.warmup):
        oracle_sample(max(64, n_sample // 4), args.n)
    vals, t_steps = [], []
    last = None
    for _ in range(args.steps):
        last = oracle_sample(n_sample, args.n)
        vals.append(1.0 / last["t_target"])
        t_steps.append(last["t_total"])
    value = statistics.mean(vals)
    sample = (f"oracle Alg. 2 at n={n_sample} (same jittered grid, theta={THETA}); generation timed and scaled "
              f"by (n/{n_sample})^2, Cholesky+solve by (n/{n_sample})^3 to n={args.n}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(t_steps), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"loglik n={args.n} theta={THETA} (BASELINE configs[2])", "n": args.n,
                   "sample_n": n_sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle", "sample": sample,
                         "extrapolated": True, "cpu_model": cpu_model(),
                         "measured_whole_evaluations": oracle_measured()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- distributed helpers
def grid_shape(spec: str, world: int):
    """P x Q process grid for `world` ranks: "PxQ" (P Q = world), or "auto": the squarest
    grid with P <= Q (1x1, 1x2, 2x2, 2x4 for 1/2/4/8 GPUs -- SURVEY §8(d) cfg 4)."""
    if spec and spec != "auto":
        P, Q = (int(v) for v in spec.lower().split("x"))
        if P * Q != world:
            raise SystemExit(f"--grid {spec}: P*Q must equal the number of ranks ({world})")
        return P, Q
    P = max(p for p in range(1, int(world**0.5) + 1) if world % p == 0)
    return P, world // P

def dist_env():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def reduce_max(value: float, dist, device: str = "cpu") -> float:
    """Max of a per-rank float over the default process group (identity without one)."""
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- side measurements
def run_extras(ex, si, torch, device: int) -> dict:
    """BASELINE configs[0], [1], [2] as side measurements (1 GPU, untimed by the driver):
    n = 400 latency, the n = 1600 MLE (nu in {0.5, 1.0}) and the n = 10k-80k sweep."""
    import math

    out = {}
    dev = f"cuda:{device}"
    with ex.Context(device=device) as c:
        # configs[0]: single evaluation at n = 400 (20 x 20 jittered grid)
        x, y = ex.gen_locations(400, SEED)
        z = c.simulate(x, y, si.normals(400, SEED), THETA)
        X, Y, Z = (torch.from_numpy(a).to(dev) for a in (x, y, z))
        for _ in range(20):
            c.loglik_dev(X, Y, Z, THETA)
        dt, walls = [], []
        for _ in range(100):
            t0 = time.perf_counter()
            r = c.loglik_dev(X, Y, Z, THETA)
            walls.append(time.perf_counter() - t0)
            dt.append(r.info["ms_total"])
        out["config1_n400"] = {"loglik": r.loglik, "device_us_median": 1e3 * statistics.median(dt),
                               "wall_us_median": 1e6 * statistics.median(walls), "kernels": r.info["kernels"]}
        # configs[1]: full MLE of (sigma2, beta, nu) at n = 1600
        lo, hi = (0.01, 0.01, 0.1), (5.0, 2.0, 2.0)
        start = tuple(math.sqrt(a * b) for a, b in zip(lo, hi))
        x, y = ex.gen_locations(1600, SEED)
        for nu in (0.5, 1.0):
            z = c.simulate(x, y, si.normals(1600, SEED), (1.0, 0.1, nu))
            # 3-D search (the paper's) / theta1 profiled out (R20); Nelder-Mead / quadratic-model
            # trust region (BOBYQA class)
            for prof in (False, True):
                for meth in ("nelder-mead", "trust-region"):
                    t0 = time.perf_counter()
                    th, ll, ne, _ = c.mle(x, y, z, lo, hi, start, xtol_rel=1e-6, max_evals=2000, profile=prof,
                                          method=meth)
                    sec = time.perf_counter() - t0
                    tag = ("_profile" if prof else "") + ("_tr" if meth == "trust-region" else "")
                    out[f"config2_mle{tag}_n1600_nu{nu}"] = {
                        "theta_hat": th, "loglik": ll, "evals": ne, "seconds": sec,
                        "ms_per_eval": 1e3 * sec / max(ne, 1)}
        # configs[2]: single-GPU sweep n = 10k - 80k (n = 100k is the headline line)
        sweep = []
        for n in (10_000, 20_000, 40_000, 60_000, 80_000):
            x, y = ex.gen_locations(n, SEED)
            zz = si.normals(n, SEED)
            X, Y, Z = (torch.from_numpy(a).to(dev) for a in (x, y, zz))
            c.loglik_dev(X, Y, Z, THETA)
            r = c.loglik_dev(X, Y, Z, THETA)
            i = r.info
            tf = n**3 / 3 / (i["ms_chol"] * 1e-3) / 1e12
            sweep.append({"n": n, "nb": i["nb"], "evals_per_s": 1e3 / i["ms_total"], "ms": i["ms_total"],
                          "phase_ms": {"gen": i["ms_gen"], "chol_and_solve": i["ms_chol"], "reduce": i["ms_reduce"]},
                          "cholesky_tflops": tf, "cholesky_frac_fp64_peak": tf / FP64_PEAK_TFLOPS,
                          "gen_gb_per_s": 8.0 * n * (n + 1) / 2 / (i["ms_gen"] * 1e-3) / 1e9,
                          "graphs": n <= 32768})
        out["config3_sweep"] = sweep
    return out


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import numpy as np
    import torch

    import paper_1708_02835_b200 as ex
    import synth_inputs as si

    rank, world, local = dist_env()
    if args.gpus != world:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nccl_id = ex.exchange_nccl_id(rank, world)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.Stream(device=local)
    # one exact evaluation distributed over all ranks (2-D block-cyclic tiles on a P x Q
    # process grid, NCCL slice broadcasts along process rows and columns): strong scaling at
    # fixed n (weak scaling: tools/scaling_sweep.sh scales n with the GPU count)
    P, Q = grid_shape(args.grid, world)
    ctx = ex.Context(device=local, stream=stream, world=world, rank=rank, nccl_id=nccl_id, grid_rows=P)
    n = args.n
    # inputs: jittered grid (Sec. 7.1) and z = L(theta) e (Alg. 1), identical on every rank -- untimed
    x, y = ex.gen_locations(n, SEED)
    e = si.normals(n, SEED)
    t0 = time.time()
    z = ctx.simulate(x, y, e, THETA)
    log(f"[rank {rank}] inputs ready (simulate {time.time() - t0:.1f}s)")
    X, Y, Z = (torch.from_numpy(a).to(f"cuda:{local}") for a in (x, y, z))
    torch.cuda.synchronize()

    # ---- device-resident arm (value) ----
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            r = ctx.loglik_dev(X, Y, Z, THETA)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    infos = []
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            r = ctx.loglik_dev(X, Y, Z, THETA)
            infos.append(r.info)
        ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms_max = reduce_max(ev0.elapsed_time(ev1), dist, f"cuda:{local}")
    ms_per_step = ms_max / args.steps
    value = args.steps / (ms_max / 1e3)  # whole-job evaluations per second

    # ---- end-to-end arm (host pointers, pinned buffers, H2D + D2H per step) ----
    hx, hy, hz = (torch.from_numpy(a).pin_memory() for a in (x, y, z))
    with torch.cuda.stream(stream):
        r_e2e = ctx.loglik(hx.numpy(), hy.numpy(), hz.numpy(), THETA)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 3))
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(e2e_steps):
            r_e2e = ctx.loglik(hx.numpy(), hy.numpy(), hz.numpy(), THETA)
        e1.record(stream)
    barrier()
    ms_e2e = reduce_max(e0.elapsed_time(e1), dist, f"cuda:{local}")
    e2e_value = e2e_steps / (ms_e2e / 1e3)

    # ---- per-evaluation breakdown and roofline of the dominant kernel ----
    # the dominant kernel gemm_nt_dmma<SyrkMap>: all its launches (bulk updates U2 on the
    # low-priority stream and lookahead updates U1 of the next panel, concurrent on the
    # high-priority stream): algorithmic flops over the union of their CUDA-event spans
    tr_ms = sum(i["ms_update_union"] for i in infos)
    tr_fl = sum(i["update_flops"] for i in infos)
    tr_n = sum(i["update_launches"] for i in infos)
    achieved = tr_fl / (tr_ms * 1e-3) / 1e12 if tr_ms > 0 else None
    u2_ms = sum(i["ms_trailing"] for i in infos)
    u2_fl = sum(i["trailing_flops"] for i in infos)
    u2_tf = u2_fl / (u2_ms * 1e-3) / 1e12 if u2_ms > 0 else None
    chol_ms = statistics.mean(i["ms_chol"] for i in infos)
    chol_tf = (n**3 / 3.0) / (chol_ms * 1e-3) / 1e12
    launches = sum(i["kernels"] for i in infos)
    traffic, traffic_of = None, None
    prof = os.path.join(ROOT, "profiles", "trailing_dram_bytes.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            traffic = tj.get("dram_bytes_per_launch")
            traffic_of = (f"{tj.get('launch')}: {tj.get('flops_per_launch', 0):.3e} algorithmic flop "
                          f"(ncu --set full, {tj.get('source')})")
        except Exception:
            traffic = None

    extras = None
    if world == 1 and not args.no_extras:
        extras = run_extras(ex, si, torch, local)

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            s = oracle_sample(args.cpu_sample, n)
            cpu = {"value": 1.0 / s["t_target"], "unit": UNIT, "cores": s["cores"], "kind": "oracle",
                   "extrapolated": True,
                   "sample": (f"oracle Alg. 2 at n={args.cpu_sample} on host cores ({s['t_total']:.1f}s: "
                              f"gen {s['t_gen']:.1f}s scaled (n/{args.cpu_sample})^2, chol+solve "
                              f"{s['t_chol']:.1f}s scaled (n/{args.cpu_sample})^3 to n={n})"),
                   "cpu_model": cpu_model(),
                   "measured_whole_evaluations": oracle_measured()}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"loglik n={n} theta={THETA} jittered grid, z=L e (BASELINE configs[2])",
                       "n": n, "nb": infos[-1]["nb"], "tiles": infos[-1]["ntiles"],
                       "parallelism": f"2-D block-cyclic {P}x{Q} process grid over {world} GPUs (NCCL)"
                       if world > 1 else "single GPU", "grid": f"{P}x{Q}",
                       "l2": "inputs (40.6 GB tiles) >> L2; no flush needed"},
            "loglik": r.loglik,
            "phase_ms": {"gen": statistics.mean(i["ms_gen"] for i in infos), "chol_and_solve": chol_ms,
                         "reduce": statistics.mean(i["ms_reduce"] for i in infos)},
            "cholesky_tflops": chol_tf,
            "cholesky_frac_fp64_peak": chol_tf / FP64_PEAK_TFLOPS,
            "cholesky_frac_cublas_dgemm": chol_tf / DGEMM_TFLOPS,
            "roofline": {"bound": "tensor",
                         "kernel": "trail_update_kernel<SyrkMap> (trailing update, CUTLASS DMMA mainloop: bulk "
                                   "U2 + lookahead U1 launches, union of their spans)",
                         "u2_only": {"achieved": u2_tf, "frac": (u2_tf / FP64_PEAK_TFLOPS) if u2_tf else None,
                                     "note": "U2 flops over U2 spans; U1 and the panel chain share the GPU "
                                             "during them"},
                         "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None,
                         "frac_vs_cublas_dgemm": (achieved / DGEMM_TFLOPS) if achieved else None,
                         "cublas_dgemm_8192_tflops": DGEMM_TFLOPS, "traffic": traffic,
                         "traffic_of": traffic_of,
                         "launches": tr_n, "share_of_step": (tr_ms / args.steps) / ms_per_step,
                         "peak_source": FP64_PEAK_SOURCE,
                         "flops_per_launch": "2*nb per (row, col) pair of the true lower triangle updated "
                                             "(+ z row), see DESIGN.md"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 3 * 8 * n,
                    "d2h_bytes_per_step": 3 * 8 + 4, "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clk,
            "other_configs": extras,
        }
        print(json.dumps(result), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--grid", default="auto", help="process grid PxQ for N > 1 GPUs (default: squarest, P <= Q)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=5000)
    ap.add_argument("--ref-sample", type=int, default=5000, help="oracle sample n of --impl reference "
                    "(the same sample as cpu_baseline, so the two CPU arms measure the same thing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip BASELINE configs 1-3 side measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
