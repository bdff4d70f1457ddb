#!/usr/bin/env python
"""Benchmark of the QTT hot path (BASELINE.json configs[1]).

One step = the isolated config-2 workload: for every (rA, rx) in
{4,8,16} x {16,64,128}: exact TT matvec y = A x (d = 24 binary cores) and
tt_round(y, 1e-10).  Inputs are seeded exactly as SURVEY.md §8(d)
(default_rng(1000+rA) for A, default_rng(2000+rx) for x, N(0,1)/sqrt(r)).
``value`` = nominal FP64 GFLOP/s over the step (matvec flops + the
reference's rounding flop count over the shapes tt_round visits, SURVEY
§8(d) formulas), with the inputs resident in HBM.

``--impl reference`` times the reference CPU algorithm (the numpy
restatement in oracle/, all host threads) on the same workload.

Launch: ``python bench.py --gpus N --steps K --warmup W`` (N>1 through
torch.distributed.run: independent replicas, one per GPU, max-over-ranks
device time; the path has no exchange step).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QTT solve wall-time at 2^10x2^10 Q1 mesh; TT matvec+round FP64 GFLOP/s vs roofline"
D = 24
EPS = 1e-10
PAIRS = [(a, b) for a in (4, 8, 16) for b in (16, 64, 128)]
CPU_SAMPLE_PAIRS = [(16, 64), (8, 128)]


# ---------------------------------------------------------------- workload


def make_inputs(rA: int, rx: int, d: int = D):
    """Seeded config-2 cores."""
    rng_a = np.random.default_rng(1000 + rA)
    ra = [1] + [rA] * (d - 1) + [1]
    A = [rng_a.standard_normal((ra[k], 2, 2, ra[k + 1])) / np.sqrt(rA) for k in range(d)]
    rng_x = np.random.default_rng(2000 + rx)
    rc = [1] + [rx] * (d - 1) + [1]
    x = [rng_x.standard_normal((rc[k], 2, rc[k + 1])) / np.sqrt(rx) for k in range(d)]
    return A, x


def qr_flops(M, N):
    return 4 * M * N * N - 4 * N**3 / 3 if M >= N else 2 * N * M * M + 2 * M**3 / 3


def svd_flops(M, N):
    mx, mn = max(M, N), min(M, N)
    return 6 * mx * mn * mn + 20 * mn**3


def round_flops(rin, rout, n=2):
    """Nominal flops over the shapes ttcore.tt_round visits."""
    d = len(rin) - 1
    r = list(rin)
    f = 0.0
    for k in range(d - 1, 0, -1):
        M, N = n * r[k + 1], r[k]
        kk = min(M, N)
        f += qr_flops(M, N) + 2 * (r[k - 1] * n) * r[k] * kk
        r[k] = kk
    for k in range(d - 1):
        f += svd_flops(r[k] * n, r[k + 1])
        f += 2 * rout[k + 1] * r[k + 1] * n * r[k + 2]
        r[k + 1] = rout[k + 1]
    return f


def expected_ranks(R, d=D):
    return [1] + [min(R, 2**k, 2 ** (d - k)) for k in range(1, d)] + [1]


def matvec_cost(rA, rx, d=D):
    ra = [1] + [rA] * (d - 1) + [1]
    rc = [1] + [rx] * (d - 1) + [1]
    flops = sum(2 * 2 * ra[l] * rc[l] * 2 * ra[l + 1] * rc[l + 1] for l in range(d))
    byts = sum(
        8 * (ra[l] * 4 * ra[l + 1] + rc[l] * 2 * rc[l + 1] + ra[l] * rc[l] * 2 * ra[l + 1] * rc[l + 1])
        for l in range(d)
    )
    return flops, byts


WORKLOAD = ("config2: TT matvec (d=24, rA in {4,8,16}, rx in {16,64,128}) + tt_round eps=1e-10, "
            "all 9 pairs per step")


def config_dict(flops):
    """The ``config`` object both arms print (identical keys and values)."""
    return {"workload": WORKLOAD, "gflop_per_step": round(flops / 1e9, 3)}


def step_flops(pairs):
    tot = 0.0
    for rA, rx in pairs:
        R = rA * rx
        tot += matvec_cost(rA, rx)[0]
        tot += round_flops([1] + [R] * (D - 1) + [1], expected_ranks(R))
    return tot


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = (
        "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
        "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
        "clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": float(max(smax)) if smax else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


# ----------------------------------------------------------------- our arm


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def job_throughput(local_ms: float, steps: int, flops_per_replica: float, dist, world: int, dev):
    """Whole-job throughput of N independent replicas: the step time is the
    MAX over ranks of the device-timed total (all_reduce MAX), the work is
    world x one replica's nominal flops.  Returns (ms_per_step, GFLOP/s)."""
    import torch

    t = torch.tensor([local_ms], dtype=torch.float64, device=dev)
    if dist is not None and world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / steps
    return ms_per_step, world * flops_per_replica / (ms_per_step * 1e-3) / 1e9


def run_ours(args):
    import torch

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_07778_b200 import _lib
    from paper_2501_07778_b200 import ttcore as T

    dev = torch.device("cuda", local)
    host = {p: make_inputs(*p) for p in PAIRS}
    resident = {p: (T.TTMatrix(host[p][0]), T.TTVector(host[p][1])) for p in PAIRS}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def pair_job(p):
        A, x = resident[p]
        return T.tt_round(T.tt_matvec(A, x), EPS)

    def one_step(check=False, serial=False):
        # the 9 pairs are independent TT problems: by default they run
        # concurrently, one stream + host thread each (latency-bound small
        # roundings overlap the GEMM-bound large ones)
        if serial or args.serial:
            zs = [pair_job(p) for p in PAIRS]
        else:
            # largest pairs first: they bound the step
            order = sorted(PAIRS, key=lambda p: -p[0] * p[1])
            zs = dict(zip(order, _lib.run_concurrent([(pair_job, p) for p in order])))
            zs = [zs[p] for p in PAIRS]
        return {p: z.ranks for p, z in zip(PAIRS, zs)} if check else {}

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (+ rank check of the rounding against the reference caps)
    for w in range(args.warmup):
        ranks = one_step(check=(w == 0))
        if w == 0:
            for (rA, rx), rk in ranks.items():
                if list(rk) != expected_ranks(rA * rx):
                    raise RuntimeError(f"rank mismatch for {rA}x{rx}: {rk}")
    flops = step_flops(PAIRS)

    clocks = ClockSampler(local)
    clocks.start()
    total_ms = 0.0
    launches0 = _lib.launch_count()
    for s in range(args.steps):
        flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_step()
        e1.record(stream)
        barrier()
        total_ms += e0.elapsed_time(e1)
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    ms_per_step, value = job_throughput(total_ms, args.steps, flops, dist, world, dev)

    # ---- end to end through the public API with host buffers
    e2e_ms = 0.0
    h2d = d2h = 0
    n_e2e = max(1, min(args.steps, 2))
    for s in range(-1, n_e2e):  # s = -1: untimed warm-up (pinned staging buffers)
        flush.zero_()
        barrier()
        t0 = time.perf_counter()

        def e2e_job(p):
            Ah, xh = host[p]
            # host=True: the rounded cores are streamed to pinned host memory while the
            # sweep runs (qtt_round_to_host); .cores are those host arrays
            z = T.tt_round(T.tt_matvec(T.TTMatrix(Ah), T.TTVector(xh)), EPS, host=True)
            e2e_out[p] = z.cores
            return z

        e2e_out = {}
        if args.serial:
            for p in PAIRS:
                e2e_job(p)
        else:
            _lib.run_concurrent([(e2e_job, p) for p in sorted(PAIRS, key=lambda p: -p[0] * p[1])])
        torch.cuda.synchronize()
        if s == 0:
            for p in PAIRS:
                Ah, xh = host[p]
                h2d += sum(c.nbytes for c in Ah) + sum(c.nbytes for c in xh)
                d2h += sum(c.nbytes for c in e2e_out[p])
        if s >= 0:
            e2e_ms += (time.perf_counter() - t0) * 1e3
    e2e_ms /= n_e2e
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * flops / (float(te.item()) * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (DMMA GEMM) from per-launch events
    barrier()
    # clean serial step (the GEMM share below is relative to it); one untimed
    # serial pass first so the main stream's allocator pool is warm
    one_step(serial=True)
    torch.cuda.synchronize()
    flush.zero_()
    barrier()
    es0 = torch.cuda.Event(enable_timing=True)
    es1 = torch.cuda.Event(enable_timing=True)
    es0.record(stream)
    one_step(serial=True)
    es1.record(stream)
    torch.cuda.synchronize()
    serial_ms = es0.elapsed_time(es1)
    _lib.gemm_profile_start()  # per-launch GEMM events: serial pass (global profiler state)
    one_step(serial=True)
    torch.cuda.synchronize()
    gflop, gms, glaunch = _lib.gemm_profile_stop()
    fp64_peak = measure_fp64_peak(torch, dev)
    achieved = gflop / (gms * 1e-3) / 1e12 if gms > 0 else 0.0

    # matvec (HBM-bound) achieved bandwidth on the largest pair, for context
    A, x = resident[(16, 128)]
    # back-to-back launches so host-side call overhead is hidden behind the
    # 250 us kernels; the 1.5 GB output of every launch exceeds L2
    mv_ms = []
    for _ in range(3):
        flush.zero_()
        T.tt_matvec(A, x)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            T.tt_matvec(A, x)
        e1.record(stream)
        torch.cuda.synchronize()
        mv_ms.append(e0.elapsed_time(e1) / 5)
    mv_bytes = matvec_cost(16, 128)[1]
    peaks = load_peaks()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample()
    extras = None
    if rank == 0 and not args.no_extras:
        extras = run_extras(torch, T, cpu_baseline=(world == 1 and not args.no_cpu_baseline))

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": config_dict(flops),
            "config_notes": {
                "pairs": "serial" if args.serial else "concurrent (one stream per pair)",
                "l2": "flushed between steps (256 MiB write); y cores up to 1.48 GB exceed L2",
                "parallelism": f"replicas x{world}",
            },
            "e2e": {
                "value": round(e2e_value, 3),
                "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
            },
            "gpu_launches": int(launches // max(args.steps, 1)) * args.steps,
            "roofline": {
                "kernel": "gemm_kernel (DMMA m8n8k4 f64) inside tt_round",
                "bound": "tensor",
                "achieved": round(achieved, 3),
                "peak": round(fp64_peak, 3),
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no FP64 entry)",
                "unit": "TFLOP/s",
                "frac": round(achieved / fp64_peak, 4) if fp64_peak else None,
                # dram__bytes_read.sum + dram__bytes_write.sum of the largest GEMM launch of the
                # step (ncu --set full, profiles/r02_kernel_evidence.txt): the 2048 x 4096 x 2048
                # carry product of the (16,128) pair, 34.4 GFLOP in 1.03 ms (33 TF/s) -- 262.5 MB read +
                # 53.6 MB written against 167.8 MB algorithmic (A, B once + C once); `achieved` is the
                # aggregate over ALL GEMM launches of the serial step, so this is per top launch
                "traffic": 316.1e6,
                "traffic_launch": {"shape": "2048x4096x2048", "gflop": 34.36, "ms": 1.033, "tflops": 33.3,
                                   "algorithmic_bytes": 167.8e6},
                "gemm_launches_per_step": int(glaunch),
                "gemm_share_of_step": round(gms / serial_ms, 4),
                "step_nominal_tflops_frac": round(value / 1e3 / fp64_peak, 4),
                "executed_gemm_gflop_per_step": round(gflop / 1e9, 3),
                "nominal_gflop_per_step": round(flops / 1e9, 3),
                "step_executed_tflops": round(gflop / (serial_ms * 1e-3) / 1e12, 3),
                "step_executed_frac": round(gflop / (serial_ms * 1e-3) / 1e12 / fp64_peak, 4),
                "note": "frac = executed-flop rate of the DMMA GEMMs (per-launch events, serial pass); "
                        "step_executed_frac = GEMM flops actually executed in one serial step / serial "
                        "step time / peak (QR panels, Jacobi and Cholesky work not counted); "
                        "step_nominal_tflops_frac = SURVEY 8(d) nominal (reference-shape) flops / "
                        "concurrent step time / peak, which exceeds 1 because the no-truncation "
                        "certificate skips SVDs the nominal count includes",
                "serial_step_ms": round(serial_ms, 3),
            },
            "matvec_roofline": {
                "bound": "hbm",
                "achieved": round(mv_bytes / (min(mv_ms) * 1e-3) / 1e9, 1),
                "peak": peaks.get("hbm_gbs"),
                "unit": "GB/s",
                "frac": round(mv_bytes / (min(mv_ms) * 1e-3) / 1e9 / peaks["hbm_gbs"], 4)
                if peaks.get("hbm_gbs") else None,
                "pair": "16x128",
                # dram__bytes_read.sum + dram__bytes_write.sum of one launch
                # (ncu --set full, profiles/r01_summary.md): 5.98 MB + 1.416 GB
                "traffic": 1.4225e9,
                "algorithmic_bytes": mv_bytes,
            },
            "clocks": clk,
            "solve_wall_s": None if not extras else {
                k: extras["solves"][k]["total_s"] for k in ("config4_d10", "config4_d10_asm1e-12", "config5_d10", "config5_d10_refined", "config4_constE_d10",
                                                           "config1_d5")
                if k in extras["solves"]},
            "cpu_baseline": cpu,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


SURVEY_C3_TTSVD_RANKS = (1, 2, 4, 5, 6, 6, 6, 6, 6, 7, 7, 9, 10, 10, 11, 13, 14, 16, 17, 19, 23, 23, 16, 8, 4, 2, 1)


def _dev_ms(torch, fn):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


UPGRADED = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3)
# config 5: same upgraded solver, tighter truncation factor, stop at the FP64
# residual floor (stall rule): ||K|| ||u|| / ||f|| ~ 1e8 at d=10
CONFIG5 = dict(UPGRADED, trunc_factor=0.05, stall_sweeps=4, max_sweeps=30)


def _conforming_error(T, u, idx, d):
    """||u - u_conf|| / ||u_conf|| against the committed conforming ground
    truth (tests/golden/conforming_c*_d*.npz), or None if absent."""
    path = os.path.join(ROOT, "tests", "golden", f"conforming_c{idx}_d{d}.npz")
    if not os.path.exists(path):
        return None
    c = np.load(path)
    uc = T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)])
    return float(T.tt_norm(T.tt_sub(u, uc)) / T.tt_norm(uc))


def _timed_build_solve(torch, T, S, build_system, idx, d, kw, assembly_eps=None):
    import time as _t

    tm = {}
    torch.cuda.synchronize()
    t0 = _t.perf_counter()
    gsys, eps = build_system(idx, d, tm, assembly_eps=assembly_eps)
    t1 = _t.perf_counter()
    res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, **kw))
    torch.cuda.synchronize()
    t2 = _t.perf_counter()
    out = {
        "solver": kw,
        "build_s": round(t1 - t0, 3), **{k: round(v, 3) for k, v in tm.items()},
        "solve_s": round(t2 - t1, 3), "total_s": round(t2 - t0, 3), "sweeps": res.sweeps,
        "residual": res.residual, "converged": res.converged, "max_rank": max(res.u.ranks),
        "K_max_rank": max(gsys.K.ranks),
    }
    return out, gsys, res


def run_extras(torch, T, cpu_baseline=True) -> dict:
    """Configs 3, 1, 4 and 5 next to the config-2 line, device-synchronised:

    * config 3: rounding (both eps) and the 2^26 TT-SVD, with the oracle port
      timed on this host in the same run;
    * solves: config 1 (reference solver path), config 4 as specified
      (variable E, upgraded AMEn -- the reference cannot reach it at d = 10,
      profiles/r02_ref_solve_c4_d6.log), config-4 geometry with constant E on
      the reference path, config 5 (L-shape) with the stall rule, each with
      the forward error against the conforming ground truth when the fixture
      exists;
    * same-run CPU solve baseline: the oracle AMEn port (local_solver
      "direct", all host threads) on config 1 and on the config-4 geometry
      with constant E at d=6, next to the device solve of the same systems;
    * a truncating rounding: config 4's Dirichlet round(D K D) (rank 1,712
      -> 117), with its nominal flops (SURVEY §8(d) formula).
    """
    import time as _t

    from paper_2501_07778_b200 import solver as S
    from paper_2501_07778_b200.configs import build_system

    out = {}
    # ---- config 3: rounding of a 16-term rank-8 sum (d=26) and TT-SVD of 2^26
    rng = np.random.default_rng(3000)
    acc = None
    host_terms = []
    for _ in range(16):
        rk = [1] + [8] * 25 + [1]
        cores = [rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(8) for k in range(26)]
        host_terms.append(cores)
        t = T.TTVector(cores)
        acc = t if acc is None else T.tt_add(acc, t)
    c3 = {}
    for eps in (1e-6, 1e-10):
        T.tt_round(acc, eps)
        r, ms = _dev_ms(torch, lambda: T.tt_round(acc, eps))
        c3[f"round_eps{eps:g}_ms"] = round(ms, 3)
        c3[f"round_eps{eps:g}_ranks_unchanged"] = r.ranks == tuple([1] + [min(128, 2**k, 2 ** (26 - k)) for k in range(1, 26)] + [1])
    n = 1 << 13
    xs = torch.arange(n, dtype=torch.float64, device="cuda") / (n - 1)
    X, Y = torch.meshgrid(xs, xs, indexing="ij")
    from paper_2501_07778_b200.assembly import _flat_ordered

    v = _flat_ordered(torch.sin(3 * X) * torch.exp(-Y) + 0.1 * torch.cos(7 * X * Y), "zorder")
    T.tt_decompose(v, 1e-8)
    tv, ms = _dev_ms(torch, lambda: T.tt_decompose(v, 1e-8))
    c3["ttsvd_2^26_ms"] = round(ms, 3)
    c3["ttsvd_ranks_equal_reference"] = tv.ranks == SURVEY_C3_TTSVD_RANKS
    c3["ttsvd_hbm_roofline_ms"] = round(4.17e9 / 6543.4e9 * 1e3, 3)
    if cpu_baseline:
        from oracle import tt as O

        host_acc = host_terms[0]
        for t in host_terms[1:]:
            host_acc = O.add(host_acc, t)
        t0 = _t.perf_counter()
        O.round_tt(host_acc, 1e-10)
        c3["cpu_round_eps1e-10_s"] = round(_t.perf_counter() - t0, 3)
        vh = v.cpu().numpy()
        t0 = _t.perf_counter()
        O.decompose_vector(vh, 1e-8)
        c3["cpu_ttsvd_s"] = round(_t.perf_counter() - t0, 3)
        c3["cpu_cores"] = os.cpu_count()
        c3["cpu_kind"] = "port (oracle/tt.py, numpy/OpenBLAS all threads)"
    del v, X, Y, xs
    out["config3"] = c3

    # ---- solves
    solves = {}
    # config4_d10 is BASELINE's literal reading (eps = 1e-8 for assembly and
    # solve); config4_d10_asm1e-12 assembles the operator accurately and
    # solves at the same eps = 1e-8: the assembly tolerance, not the solver,
    # sets the forward error on this operator (profiles/r02_c4_error_probe.log)
    runs = (("config1_d5", 1, 5, dict(local_solver="direct"), None),
            ("config4_d10", 4, 10, UPGRADED, None),
            ("config4_d10_asm1e-12", 4, 10, UPGRADED, 1e-12),
            ("config4_constE_d10", 40, 10, dict(local_solver="direct"), None),
            ("config5_d10", 5, 10, CONFIG5, None),
            ("config5_d10_refined", 5, 10, dict(CONFIG5, refine_steps=1), None))
    saved_bits = S._DENSE_RESIDUAL_BITS
    for name, idx, d, kw, asm_eps in runs:
        if idx == 5:
            S._DENSE_RESIDUAL_BITS = 23  # 2^23 dense residual
        try:
            rec, gsys, res = _timed_build_solve(torch, T, S, build_system, idx, d, kw, asm_eps)
        finally:
            S._DENSE_RESIDUAL_BITS = saved_bits
        if asm_eps is not None:
            rec["assembly_eps"] = asm_eps
        rec["conforming_rel_error"] = _conforming_error(T, res.u, idx, d)
        solves[name] = rec
        del gsys, res
        _release(torch)
    solves["reference_cpu_s_survey"] = {
        "config1_d5_solve": 1.21, "config4_constE_d10_solve": 658.9, "config4_constE_d10_assembly": 11.05,
        "config4_d10_assembly": 43.0, "config4_d10_couple_dirichlet": 18.0,
        "note": "SURVEY Appendix B (8-core Xeon); on config 4 as specified (variable E) the reference's default "
                "solver diverges and its direct-local-solve path converges at d = 6 in 246 s with full ranks "
                "(profiles/r02_ref_solve_c4_d6.log) but cannot factor the dense local systems of d = 10"}
    if cpu_baseline:
        from oracle import amen

        same = {}
        for name, idx, d in (("config1_d5", 1, 5), ("config4_constE_d6", 40, 6)):
            gsys, eps = build_system(idx, d)
            K = list(gsys.K.cores)  # host numpy copies
            f = list(gsys.f.cores)
            t0 = _t.perf_counter()
            r = amen.solve(K, f, eps=eps, seed=0)
            cpu_s = _t.perf_counter() - t0
            torch.cuda.synchronize()
            t0 = _t.perf_counter()
            g = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver="direct"))
            torch.cuda.synchronize()
            gpu_s = _t.perf_counter() - t0
            same[name] = {"cpu_solve_s": round(cpu_s, 3), "cpu_sweeps": r["sweeps"],
                          "cpu_residual": r["residual"], "gpu_solve_s": round(gpu_s, 3),
                          "gpu_sweeps": g.sweeps, "gpu_residual": g.residual,
                          "speedup": round(cpu_s / gpu_s, 1)}
        same["cores"] = os.cpu_count()
        same["kind"] = "port (oracle/amen.py: reference AMEn restated, local_solver='direct', OpenBLAS all threads)"
        solves["same_run_cpu_solve"] = same
    out["solves"] = solves

    # ---- a truncating rounding: config 4's Dirichlet round(D K D)
    from paper_2501_07778_b200.assembly import assemble_subdomain
    from paper_2501_07778_b200.configs import config
    from paper_2501_07778_b200.coupling import concat_blocks
    from paper_2501_07778_b200.topology import DomainTopology

    meshes, mat, body, eps = config(4, 10)
    systems = [assemble_subdomain(m, mat, "zorder", eps, body_force=body) for m in meshes]
    g = concat_blocks(systems, DomainTopology.from_subdomains(meshes), ordering="zorder", epsilon=eps)
    dmask = T.tt_diag(g.mask)
    dkd = T.tt_matmat(dmask, T.tt_matmat(g.K, dmask))
    T.tt_round(dkd, eps)
    kr, ms = _dev_ms(torch, lambda: T.tt_round(dkd, eps))
    nominal = round_flops(list(dkd.ranks), list(kr.ranks), n=4)
    out["dirichlet_round"] = {
        "ms": round(ms, 3), "pre_round_max_rank": max(dkd.ranks), "out_max_rank": max(kr.ranks),
        "nominal_gflop": round(nominal / 1e9, 2),
        "nominal_tflops": round(nominal / (ms * 1e-3) / 1e12, 3),
        "note": "truncating rounding (one-sided Jacobi path); nominal = SURVEY 8(d) QR + R-SVD count over the "
                "shapes tt_round visits"}
    return out


def _release(torch):
    try:
        from paper_2501_07778_b200 import _lib

        _lib.release_cached()
    except Exception:
        torch.cuda.empty_cache()


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback B200_PROFILING.md"}


def measure_fp64_peak(torch, dev) -> float:
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b
    return 2 * n**3 / best / 1e12


# ----------------------------------------------------- CPU reference timing


def _cpu_step(pairs, inputs):
    from oracle import tt as O

    for p in pairs:
        A, x = inputs[p]
        O.round_tt(O.matvec(A, x), EPS)


def cpu_baseline_sample() -> dict:
    """Reference algorithm (numpy restatement, all host threads) on a bounded
    sample of the same workload: the (16,64) and (8,128) pairs."""
    inputs = {p: make_inputs(*p) for p in CPU_SAMPLE_PAIRS}
    t0 = time.perf_counter()
    _cpu_step(CPU_SAMPLE_PAIRS, inputs)
    dt = time.perf_counter() - t0
    return {
        "value": round(step_flops(CPU_SAMPLE_PAIRS) / dt / 1e9, 3),
        "unit": "GFLOP/s",
        "cores": os.cpu_count(),
        "kind": "port",
        "sample": "matvec+round(1e-10) of the (16,64) and (8,128) config-2 pairs, numpy/OpenBLAS all threads",
        "seconds": round(dt, 2),
    }


def run_reference(args):
    world, rank, local = _dist_env()
    if rank != 0:
        return
    inputs = {p: make_inputs(*p) for p in PAIRS}
    # warm-up on the smallest pair only (numpy has no JIT; keeps the run bounded)
    for _ in range(args.warmup):
        _cpu_step([(4, 16)], inputs)
    flops = step_flops(PAIRS)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _cpu_step(PAIRS, inputs)
    dt = time.perf_counter() - t0
    value = flops * args.steps / dt / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": config_dict(flops),
        "cpu_baseline": {
            "value": round(value, 3),
            "unit": "GFLOP/s",
            "cores": os.cpu_count(),
            "kind": "port",
            "sample": "full config-2 sweep per step; reference algorithm restated in numpy (oracle/tt.py), OpenBLAS all threads",
        },
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--serial", action="store_true", help="run the 9 config-2 pairs one after another")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
