#!/usr/bin/env python
"""Benchmark of the matrix-free K_y.V hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg4]

One *step* = one (K + noise I) V product over the whole synthetic workload of
the config (default cfg4: RBF(0.5), N=100,000, D=8, V = the t=16 SLQ probe
vectors), with X and V resident in HBM. Under torchrun (N>1) the rows of K are
sharded over the ranks and each step ends with the library's NCCL all-gather
of the product slices, so every rank holds the full product (strong scaling:
total work fixed). Device time per step from CUDA events on the library's
stream, L2 flushed (256 MiB memset) before every timed step, summed over the
K steps, max over ranks.

Also reported: `e2e` (the same metric through the public Python API with
pinned host buffers, H2D of X and V and D2H of the product inside the timed
region), the CG solve time (t=1 alpha solve, tol 1e-8, max_iter min(N,1000))
and the SLQ log-det time (16 probes x 50 Lanczos steps), the roofline of the
fused K1 kernel (per-launch CUDA events) and the CPU baseline (the pinned
oracle port of the reference, rank 0 only).

`--impl reference` times the reference's own CPU algorithm (oracle port of
minigp's matrix_free_matvec; the reference is pure Python) on a bounded row
sample of the same workload per step, on rank 0 only.
"""

from __future__ import annotations

import argparse
import contextlib
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kernel-matvec Gentries/s and CG solve time at N=100k, D=8, 1/2/4/8 B200"
UNIT = "Gentries/s"
SM_COUNT = 148
FP32_LANES = 128
SFU_PER_SM = 16  # MUFU.EX2 per clock per SM: tools/alu_bench.cu measures 15.96, ncu
                 # sm__inst_executed_pipe_xu 99.6 % (profiles/r02_alu_mufu_ncu.txt)


DTYPE_TC = ("f32 kernel entries from an FP16x2-split tcgen05 distance GEMM (FP32 accumulate) and "
            "MUFU exp2; contraction on tcgen05 with FP16 hi/lo entries x FP16 hi/lo V (power-of-two "
            "column scaling), FP32 TMEM accumulation over 1024-column groups, f64 sums")


def tc_rhs_per_pass(t):
    """Right-hand sides per K1-TC pass (lgp_codegen.cpp make_tc_plan)."""
    return 8 if t <= 8 else (16 if t <= 16 else (32 if t <= 32 else 64))


def flops_per_entry(kernel_expr, d, t):
    """Algorithmic work per kernel entry: distance 3D, leaf
    transform, +2t for the contraction. Transcendentals are SFU ops, not flops."""
    if kernel_expr.startswith("(rbf"):
        return 3 * d + 1 + 2 * t, 1
    if kernel_expr.startswith("(matern52"):
        return 3 * d + 5 + 2 * t, 2
    if kernel_expr.startswith("(matern32"):
        return 3 * d + 3 + 2 * t, 2
    if kernel_expr.startswith("(+ (scale 1.0 (rbf"):  # cfg3 composite
        return 3 * d + 1 + 4 * d + 1 + 3 + 2 * t, 2 + d
    return 3 * d + 2 * t, 1


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnosis only: no sampler process
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a few hundred ms to start: wait for its first
            # sample so the (short) timed region is covered
            t_wait = time.time() + 5.0
            while not self.lines and time.time() < t_wait and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self, which):
        """Wall-clock bounds of the timed region (samples are filtered to it)."""
        setattr(self, which, time.time())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        t0, t1 = getattr(self, "t_start", None), getattr(self, "t_end", None)
        inside = [r for r in rows if t0 is None or (t0 - 0.03 <= r[0] <= t1 + 0.03)]
        if len(inside) < 3 and rows and t0 is not None:  # short region: nearest samples
            mid = 0.5 * (t0 + t1)
            inside = sorted(rows, key=lambda r: abs(r[0] - mid))[:3]
        reasons = set()
        for r in inside:
            for nm, val in zip(names, r[3]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        sm = [r[1] for r in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(r[2] for r in inside) if inside else None,
                "samples": len(sm),
                "reasons": sorted(reasons)}


@contextlib.contextmanager
def stdout_to_stderr():
    """Route file descriptor 1 to stderr (native libraries printing at init)."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def max_over_ranks(ctx, value):
    """Max of a host value over the ranks (the library's NCCL all-reduce; no
    torch.distributed). Identity at one rank."""
    if ctx is None or ctx.world == 1:
        return value
    return ctx.allreduce_max([value])[0]


def host_info():
    """CPU model, core count and the BLAS thread pools (threadpoolctl)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    pools = []
    try:
        import threadpoolctl

        pools = [{"api": i.get("internal_api"), "version": i.get("version"),
                  "num_threads": i.get("num_threads")} for i in threadpoolctl.threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "threadpools": pools}


def cpu_baseline(cfg, x, seconds=12.0, cg_iterations=None):
    """Oracle port of the reference matvec (block=32 fit path, one RHS column)
    on a row subset of the same workload; extrapolated as entries/s, and the
    CPU CG solve time extrapolated as (time of one full matvec) x iterations
    (SURVEY.md §8d)."""
    from oracle import gp_oracle as O

    nodes = O.parse_tree(cfg["kernel"])
    v = np.random.default_rng(1).standard_normal(cfg["n"])
    rows = 1024 if cfg["n"] >= 50_000 else min(cfg["n"], 4096)
    done, elapsed, reps = 0, 0.0, 0
    while elapsed < seconds or reps < 2:
        r0 = (reps * rows) % max(cfg["n"] - rows, 1)
        t0 = time.perf_counter()
        O.matvec(nodes, x, cfg["noise"], v, block=32, row_range=(r0, r0 + rows))
        elapsed += time.perf_counter() - t0
        done += rows * cfg["n"]
        reps += 1
    info = host_info()
    threads = max([p["num_threads"] or 1 for p in info["threadpools"]] or [os.cpu_count() or 1])
    rate = done / elapsed  # entries / s, one RHS column
    out = {"value": rate / 1e9, "unit": UNIT, "cores": int(threads), "kind": "port",
           "sample": f"{reps} x {rows}-row slabs x all {cfg['n']} columns, t=1 (reference has no "
                     f"multi-RHS path: t columns cost t x), block=32, FP64 NumPy/OpenBLAS "
                     f"({threads} BLAS threads, ufuncs single-threaded), {elapsed:.1f} s",
           "matvec_s_extrapolated": cfg["n"] ** 2 / rate}
    out.update(info)
    if cg_iterations:
        out["cg_solve_s_extrapolated"] = cg_iterations * cfg["n"] ** 2 / rate
        out["cg_solve_note"] = (f"one full reference matvec ({cfg['n'] ** 2 / rate:.1f} s) x the "
                                f"{cg_iterations} iterations of the device solve")
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference CPU algorithm (oracle port), rank 0 only."""
    if rank != 0:
        return 0
    from oracle import gp_oracle as O

    cfg = dict(O.CONFIGS[args.config])
    x, _ = O.synthetic(cfg["n"], cfg["d"])
    t = cfg["t"]
    z = O.probes(cfg["n"], t)
    nodes = O.parse_tree(cfg["kernel"])
    rows = 64 if cfg["n"] >= 50_000 else min(cfg["n"], 512)
    times = []
    # rank 0 runs alone: give the BLAS all host cores (torchrun sets OMP_NUM_THREADS=1)
    try:
        import threadpoolctl

        limiter = threadpoolctl.threadpool_limits(limits=os.cpu_count())
    except Exception:
        limiter = None
    for s in range(args.warmup + args.steps):
        r0 = (s * 997 * rows) % max(cfg["n"] - rows, 1)
        t0 = time.perf_counter()
        O.matvec(nodes, x, cfg["noise"], z, block=32, row_range=(r0, r0 + rows))
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = args.steps * rows * cfg["n"] * t / total / 1e9
    info = host_info()
    threads = max([p["num_threads"] or 1 for p in info["threadpools"]] or [os.cpu_count() or 1])
    sample = (f"per step: {rows}-row slab of the {cfg['n']}x{cfg['n']} operator x {t} RHS columns "
              f"(each column a separate reference matvec, block=32)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, cfg),
            "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": int(threads), "kind": "port",
                                  "sample": sample}, **info),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name, cfg, world=1, sharded=False):
    par = (f"row-sharded K over {world} rank(s), NCCL all-gather" if (world > 1 or sharded)
           else "one GPU (all rows of K)")
    return {"workload": f"{name}: (K+{cfg['noise']}I)V, kernel {cfg['kernel']}, N={cfg['n']}, "
                        f"D={cfg['d']}, t={cfg['t']} SLQ probe vectors",
            "n": cfg["n"], "d": cfg["d"], "t": cfg["t"], "kernel": cfg["kernel"],
            "noise": cfg["noise"], "parallelism": par,
            "l2": "flushed (256 MiB memset) before every timed step"}


def run_ours(args, rank, world):
    import ctypes as C

    import paper_2605_17898_b200 as G
    from paper_2605_17898_b200 import _lib, distributed
    from oracle import gp_oracle as O  # input recipe + CPU baseline only

    # rank 0 prints exactly one JSON line on stdout: NCCL's own log lines
    # (communicator set-up with nranks / transports at INFO) go to stderr
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    with stdout_to_stderr():
        ctx = distributed.init(force_comm=args.sharded) if (world > 1 or args.sharded) \
            else _lib.default_context()
    dist = ctx if world > 1 else None
    lib = _lib.lib()
    cfg = dict(O.CONFIGS[args.config])
    n, d, t = cfg["n"], cfg["d"], cfg["t"]
    x, y = O.synthetic(n, d)
    z = np.ascontiguousarray(O.probes(n, t))
    kernel = G.parse_kernel(cfg["kernel"])
    prog = G.kernels.program(kernel)
    pts = _lib.DevicePoints(ctx, x)
    dv, do = C.c_void_p(), C.c_void_p()
    _lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(dv)))
    _lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(do)))
    _lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(z), z.nbytes))

    def step():
        _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, cfg["noise"],
                                  dv, t, do, _lib.DEVICE_PTRS))

    ctx.set_profile(True)
    clocks = ClockSampler(ctx.device)  # started before the warm-up: start-up latency
    clocks.start()
    for _ in range(args.warmup):
        ctx.flush_l2()
        step()
    ctx.k1_profile(reset=True)
    if dist:
        dist.barrier()
    ctx.sync()
    clocks.mark("t_start")
    launches0 = ctx.launches()
    total_ms = 0.0
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.timer_start()
        step()
        total_ms += ctx.timer_stop()
    launches = ctx.launches() - launches0
    ctx.sync()
    clocks.mark("t_end")
    if dist:
        dist.barrier()
    k1_ms, k1_n = ctx.k1_profile(reset=True)
    clk = clocks.stop()  # the clock record covers the timed region of `value`
    total_ms = max_over_ranks(dist, total_ms)
    value = n * n * t * args.steps / (total_ms * 1e-3) / 1e9

    # parity spot check of the timed product (rows owned by rank 0), vs the oracle
    out = np.empty_like(z)
    _lib.check(lib.lgp_memcpy_d2h(ctx.handle, _lib.vptr(out), do, z.nbytes))
    r0 = n // 2
    want = O.matvec(O.parse_tree(cfg["kernel"]), x, cfg["noise"], z[:, :2], block=32,
                    row_range=(r0, r0 + 64))
    parity = float(np.linalg.norm(out[r0:r0 + 64, :2] - want) / np.linalg.norm(want))

    # e2e: the public API call exactly as a NumPy caller makes it - ordinary
    # (pageable) NumPy arrays X, V in, a NumPy array out: H2D of X and V and
    # D2H of the product inside the timed region
    px = np.array(x, copy=True)
    pv = np.array(z, copy=True)
    # warm-up in the timed loop's own pattern (the previous result stays alive
    # while the next call runs), so pooled host/device buffers are in place; the
    # host-side call time settles over ~20-30 calls on the gpurun boxes
    # (tools/e2e_dist.py: 6.2 ms on call 1 -> 4.8 ms by call 20), hence 30
    for _ in range(max(30, args.warmup)):
        res = G.matrix_free_matvec(kernel, px, cfg["noise"], pv)
    if dist:
        dist.barrier()
    e2e_steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = G.matrix_free_matvec(kernel, px, cfg["noise"], pv)
    e2e_s = max_over_ranks(dist, time.perf_counter() - t0)
    del res
    e2e = {"value": n * n * t * e2e_steps / e2e_s / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": int(x.nbytes + z.nbytes), "d2h_bytes_per_step": int(z.nbytes),
           "ms_per_step": e2e_s / e2e_steps * 1e3, "host_buffers": "pageable NumPy arrays",
           "path": "paper_2605_17898_b200.matrix_free_matvec(kernel, X, noise, V) -> lgp_matvec"}

    # CG solve (alpha) and SLQ log-det through the device solver loops
    solve = {}
    if not args.no_solve:
        op = G.KernelOperator(kernel, x, cfg["noise"], ctx=ctx)
        # warm-up: JIT modules / scratch of the t = 1 CG kernels and the SLQ block
        op.cg(y, 1e-8, 2)
        op.lanczos(G.probe_block(n, t if t > 1 else 16, 0), 50)  # full-size basis scratch
        ctx.k1_profile(reset=True)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        xs, iters, resid = op.cg(y, 1e-8, None)
        cg_s = max_over_ranks(dist, time.perf_counter() - t0)
        k1_cg_ms, k1_cg_n = ctx.k1_profile(reset=True)
        t0 = time.perf_counter()
        ld = G.slq_logdet(op, n, G.CgConfig(probes=t if t > 1 else 16, lanczos_steps=50), seed=0)
        slq_s = max_over_ranks(dist, time.perf_counter() - t0)
        k1_slq_ms, k1_slq_n = ctx.k1_profile(reset=True)
        solve = {"cg_solve": {"ms": cg_s * 1e3, "iterations": int(iters[0]),
                              "final_residual": float(resid[0]), "rel_tolerance": 1e-8,
                              "k1_ms_per_matvec": k1_cg_ms / max(k1_cg_n, 1)},
                 "slq_logdet": {"ms": slq_s * 1e3, "probes": t if t > 1 else 16,
                                "lanczos_steps": 50, "logdet": ld,
                                "k1_ms_per_step": k1_slq_ms / max(k1_slq_n, 1)}}

    if rank != 0:
        return 0
    pk = measured_peaks()
    f_mhz = float(pk.get("sm_max_mhz", 1965.0))
    fp32_peak = 2 * FP32_LANES * SM_COUNT * f_mhz * 1e6 / 1e12  # TFLOP/s
    flops, sfu = flops_per_entry(cfg["kernel"], d, t)
    k1_avg_ms = k1_ms / max(k1_n, 1)
    rows_local = -(-n // world)
    achieved = rows_local * n * flops / (k1_avg_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(args.config)
    except Exception:
        pass
    tc = "lgp_matvec_tc(" in prog.source(d, t)
    sfu_peak = SFU_PER_SM * SM_COUNT * f_mhz * 1e6 / 1e12  # T op/s
    # algorithmic SFU ops per launch: one per kernel entry
    # (K1-TC re-evaluates the entries per pass of <= 32 RHS: t <= 32 is one pass)
    sfu_ach = rows_local * n * sfu / (k1_avg_ms * 1e-3) / 1e12
    bf16 = float(pk.get("bf16_tflops", 1648.7))
    if tc:
        # K1-TC: per 128 x 64 chunk the distance GEMM (K = 3D+4 rounded to 16)
        # and the contraction (K = 2 x 64, N = 2 x RHS; 64 RHS: 3 x K = 64, N = RHS) on tcgen05
        n_pass = -(-t // tc_rhs_per_pass(t))
        kh = -(-(3 * d + 4) // 16) * 16
        chunks = -(-rows_local // 128) * -(-n // 64) * n_pass
        rhs = tc_rhs_per_pass(t)
        tflop = chunks * (2 * 128 * 64 * kh + (3 * 2 * 128 * rhs * 64 if rhs == 64 else 2 * 128 * 2 * rhs * 128)) \
            / (k1_avg_ms * 1e-3) / 1e12
        roofline = {"bound": "sfu", "achieved": sfu_ach, "peak": sfu_peak, "unit": "T SFU op/s",
                    "frac": sfu_ach / sfu_peak, "traffic": traffic,
                    "kernel": "lgp_matvec_tc (fused K1: tcgen05 FP16x2 distance GEMM -> TMEM -> "
                              "exp2 epilogue -> FP16 hi/lo contraction GEMM)",
                    "k1_ms_per_launch": k1_avg_ms,
                    "resource": "the special-function unit: one exp2 per kernel entry (SURVEY.md "
                                "§8d: 1 SFU op per RBF entry), MUFU.EX2 at 16/clk/SM",
                    "peak_source": f"{SFU_PER_SM} MUFU.EX2/clk/SM x {SM_COUNT} SMs x {f_mhz:.0f} MHz: "
                                   "tools/alu_bench.cu measures 15.96/clk/SM at ncu "
                                   "sm__inst_executed_pipe_xu 99.6 %; K1-TC runs that pipe at 71.5 % "
                                   "(profiles/r02_k1tc_t16_ncu_summary.txt)",
                    "tensor": {"issued_tflops": tflop, "peak_measured_bf16_tflops": bf16,
                               "frac": tflop / bf16},
                    "algorithmic_fp32": {"flops_per_entry": flops, "tflops": achieved,
                                         "frac_of_measured_bf16": achieved / bf16,
                                         "frac_of_fp32_simt_peak": achieved / fp32_peak},
                    "hbm_frac": (traffic / (k1_avg_ms * 1e-3) / 1e9 / float(pk.get("hbm_gbs", 6444.7))
                                 if traffic else None)}
    else:
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": traffic,
                    "kernel": "lgp_matvec (fused K1, SIMT FP32/FP64)",
                    "k1_ms_per_launch": k1_avg_ms,
                    "flops_per_entry": flops, "sfu_per_entry": sfu,
                    "peak_source": f"derived: 2 x {FP32_LANES} FP32 lanes x {SM_COUNT} SMs x "
                                   f"{f_mhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)",
                    "sfu_frac": sfu_ach / sfu_peak}
        if clk.get("sm_mhz"):
            roofline["frac_at_observed_clock"] = achieved / (fp32_peak * clk["sm_mhz"] / f_mhz)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": DTYPE_TC if tc else "f32 entries, f64 accumulation (SIMT)", "data": "synthetic",
            "config": workload_config(args.config, cfg, world, args.sharded),
            "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "parity_rel_l2": parity}
    line.update(solve)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(
            cfg, x, cg_iterations=solve.get("cg_solve", {}).get("iterations"))
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="row-sharded schedule with an NCCL communicator even at one rank "
                         "(exercises the multi-GPU path on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if launched and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks",
              file=sys.stderr)
        return 2
    if args.impl == "reference":
        # the reference is a CPU algorithm: rank 0 alone runs it (other ranks exit 0)
        return run_reference(args, rank, args.gpus)
    if not launched and args.gpus > 1:
        return self_launch(args)
    return run_ours(args, rank, world)


def self_launch(args):
    """`bench.py --gpus N` without a launcher: start N ranks (one process per
    GPU) ourselves, sharing an NCCL id made here (no torch.distributed)."""
    from paper_2605_17898_b200 import _lib, distributed

    have = _lib.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
              file=sys.stderr)
        return 2
    return distributed.launch([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                              args.gpus)


if __name__ == "__main__":
    sys.exit(main())
