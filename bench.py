"""bench.py -- LR-SPIKE preconditioned solve on B200 (BASELINE.json metric).

Workload (one "step"): BASELINE.json configs[2] = c3 at P = 64 -- the largest config
that fits one GPU, the one BASELINE.md section 2 / SURVEY.md D7 quote the time-to-
tolerance target on: the 96^3 27-point heterogeneous-diffusion system (n = 884,736,
23.4M nnz, half-bandwidth 9,313, coefficients 10^U[-2,2]), 64 partitions, n_svd = 32,
GMRES(50) to 1e-8: factorize (tiled band LU of the 64 blocks + randomized spike SVDs +
truncated preconditioner) followed by the preconditioned GMRES solve.  metric =
time-to-tolerance in seconds (factorize + solve), lower is better.  `--config c2` runs
the c2 line of round 1 (P = 8, BiCGStab).

  value       device time of one step with the matrix and RHS already resident
              in HBM (CUDA events on the library stream, max over ranks)
  e2e         the same step through the public C-ABI with HOST buffers: CSR
              upload (validate + transpose + H2D), factorize, solve with a host
              RHS, x copied back -- host<->device copies inside the timed region
  roofline    the dominant kernel class of the step by CUDA-event time (c3: the
              preconditioner apply's one-RHS band sweeps, HBM-bound), with its DRAM
              traffic from the committed ncu capture (profiles/ncu_traffic.json);
              roofline_lu_update = the bulk trailing update of the band LU (the
              INT8-sliced tcgen05 kernel, or the DMMA GEMM with LRS_LU_I8=0)
  cpu_baseline the oracle port (scipy/OpenBLAS LAPACK) on the box's host cores: a
              bounded, measured sample of the same workload (one diagonal block
              factored, its spikes, 16 concurrent block solves) scaled by the exact
              partition / apply counts, beside the committed measured full run
              (tests/golden/<cfg>.json)

Multi-GPU (torchrun, one rank per GPU, NCCL): the same job with its P partitions
sharded across the ranks (lrs_factorize_dist): strong scaling, the value is the max
over ranks of the device time of one step.

--impl reference times the reference algorithm's CPU implementation (the oracle
port; the reference itself cannot be built) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

I8_PRODUCTS = 28  # digit-slice products per K chunk of the INT8 update (I8_PRODUCTS, csrc/lu_i8.cu)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = max(mx, float(f[2]))
                except ValueError:
                    continue
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                    "sw_power_cap"), f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        except Exception:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# CPU baseline (oracle port, bounded sample, extrapolated by algorithmic work)
# ---------------------------------------------------------------------------------------
def _lu_flops(n, kl, ku):
    j = np.arange(n, dtype=np.float64)
    rem = n - 1 - j
    a = np.minimum(kl, rem)
    b = np.minimum(ku, rem)
    return float(np.sum(a + 2 * a * b)), float(np.sum(a + 1 + b))


WORKLOADS = {
    "c2": ("BASELINE.json configs[1]: 64^3 7-pt convection-diffusion, n=262,144, k=4,096, P=8, "
           "n_svd=16, BiCGStab to 1e-8"),
    "c3": ("BASELINE.json configs[2] (at P=64: the largest single-GPU config, BASELINE.md 2 / "
           "SURVEY D7): 96^3 27-pt heterogeneous diffusion, n=884,736, nnz=23.4M, k=9,313, "
           "n_svd=32, GMRES(50) to 1e-8"),
    "c5": ("BASELINE.json configs[4]: FEAST contour system z_j I - A, 80^3 7-pt + symmetric "
           "perturbation, complex128, n=512,000, k=6,400, P=16, n_svd=32, 16 RHS, GMRES(40) to "
           "1e-10; one shift per rank (replicas, PAPER.md:1628)"),
}
DEFAULT_P = {"c2": None, "c3": 64, "c5": 16}


def _workload(name, P, scale):
    w = WORKLOADS.get(name, f"BASELINE config {name}")
    if scale != 1.0:
        w += f" (scaled x{scale:g})"
    return f"{name}: {w}; factorize + solve" + ("" if P is None else f" [P={P}]")


def _full_run(name, P, scale):
    """The committed measured full oracle run of this config (tests/golden/make_full_fixtures.py),
    if one exists: {t_factorize_s, t_solve_s, iterations, host}."""
    tag = f"full_{name}" if (scale == 1.0 and P is None) else f"{name}_s{scale:g}_P{P}"
    try:
        with open(os.path.join(ROOT, "tests", "golden", f"{tag}.json")) as fh:
            m = json.load(fh)
    except OSError:
        return None
    return {"fixture": f"tests/golden/{tag}.json", "t_factorize_s": m["t_factorize_s"],
            "t_solve_s": m["t_solve_s"], "value": m["t_factorize_s"] + m["t_solve_s"],
            "iterations": m["iterations"], "precond_applications": m["precond_applications"],
            "host": m.get("host")}


class _CpuSampler:
    """Bounded, measured CPU sample of the workload with the oracle (scipy/OpenBLAS LAPACK),
    run on the schedule of the oracle's own partition-parallel full run
    (LRS_ORACLE_THREADS = host threads, OPENBLAS_NUM_THREADS = 1; tests/golden/<cfg>.json).

    One sample = one WAVE of that schedule: `conc` forked single-threaded workers (one per
    host thread) each take partition i (i cycles from sample to sample; the partitions have
    the same size and structure) and
      t_fact  factor it (dgetrf / dgbtrf) and build its spikes (randomized_spike_svd of its
              T and W sides) -- the wall time of the wave, barrier to last finish
      t_ap    one one-column block solve against that factor -- wall time of the wave
    plus one CSR SpMV of the whole matrix (scipy).  Scaled by the exact counts of the
    measured GPU solve:
      T = ceil(P / conc) (t_fact + applies t_ap) + matvecs t_spmv
    (the Krylov vector operations and the r x r interface algebra are left out, which
    favours the CPU; the committed full run is reported beside it)."""

    def __init__(self, name, scale, P, threads=None):
        self.threads = threads or len(os.sched_getaffinity(0)) or os.cpu_count() or 1
        from oracle import lrspike_oracle as O  # the checker / baseline, never the product
        from paper_2504_11167_b200 import configs

        self.O = O
        self.cfg = configs.make_config(name, scale, P)
        self.S = self.cfg.matrix.to_scipy()
        self.lay = O.make_layout(self.S.shape[0], self.cfg.P, self.cfg.b)
        self.blocks = O.extract_blocks(self.S, self.lay)
        self.name, self.scale = name, scale
        self.conc = min(self.threads, self.cfg.P)
        self.i = 0

    def _wave(self, i):
        import multiprocessing as mp

        O, cfg, blocks = self.O, self.cfg, self.blocks
        os_ = (cfg.r + 1) // 2
        ctl = _openblas_threads_ctl()
        old = ctl(1) if ctl else None
        try:
            mctx = mp.get_context("fork")
            b1, b2 = mctx.Barrier(self.conc + 1), mctx.Barrier(self.conc + 1)
            q1, q2 = mctx.Queue(), mctx.Queue()

            def worker():
                b1.wait()
                fo = O.factorize_block(blocks.A[i])
                if i + 1 < cfg.P:
                    O.randomized_spike_svd(fo, blocks.B[i], O.SIDE_T, cfg.r, os_, 2, cfg.seed, i)
                if i > 0:
                    O.randomized_spike_svd(fo, blocks.C[i], O.SIDE_W, cfg.r, os_, 2, cfg.seed, i)
                q1.put(time.perf_counter())
                rhs = np.asfortranarray(np.random.default_rng(i).uniform(-1, 1, (fo.n, 1)))
                b2.wait()
                O.solve_block(fo, rhs)
                q2.put(time.perf_counter())

            procs = [mctx.Process(target=worker) for _ in range(self.conc)]
            for pr in procs:
                pr.start()
            b1.wait()
            t0 = time.perf_counter()
            t_fact = max(q1.get() for _ in procs) - t0
            b2.wait()
            t1 = time.perf_counter()
            t_ap = max(q2.get() for _ in procs) - t1
            for pr in procs:
                pr.join()
            return t_fact, t_ap
        finally:
            if ctl and old:
                ctl(old)

    def sample(self, applies, matvecs):
        cfg, i = self.cfg, self.i % self.cfg.P
        self.i += 1
        t_fact, t_ap = self._wave(i)
        x = np.ones(self.S.shape[0])
        t0 = time.perf_counter()
        self.S @ x
        t_spmv = time.perf_counter() - t0
        waves = -(-cfg.P // self.conc)
        est_f = waves * t_fact
        est_s = applies * waves * t_ap + matvecs * t_spmv
        return {"value": est_f + est_s, "t_fact_wave_s": t_fact, "t_apply_wave_s": t_ap,
                "t_spmv_s": t_spmv, "partition": i, "est_factorize_s": est_f,
                "est_solve_s": est_s}

    def describe(self, applies, matvecs):
        c = self.cfg
        waves = -(-c.P // self.conc)
        return (f"oracle (scipy OpenBLAS LAPACK) on {self.conc} host cores, the oracle's own "
                f"partition-parallel schedule (one single-threaded worker per core): per step one "
                f"wave of {self.conc} diagonal blocks of {self.name} (n_i={self.lay.sizes[0]}, "
                f"k={c.b}) factored with their spikes, then one concurrent one-column solve each; "
                f"scaled to {waves} waves x (factorization + {applies} applies) and {matvecs} "
                f"SpMVs of the measured solve")


def _openblas_threads_ctl():
    """openblas_set_num_threads of scipy's bundled OpenBLAS (ctypes), or None."""
    import ctypes
    import glob

    try:
        import scipy

        libs = glob.glob(os.path.join(os.path.dirname(scipy.__file__) + ".libs", "libscipy_openblas*.so"))
        if not libs:
            return None
        lib = ctypes.CDLL(libs[0])
        for pre in ("scipy_openblas_", "openblas_", "scipy_"):
            get = getattr(lib, pre + "get_num_threads", None) or getattr(lib, pre + "get_num_threads64_", None)
            setf = getattr(lib, pre + "set_num_threads", None) or getattr(lib, pre + "set_num_threads64_", None)
            if get and setf:
                def ctl(n, get=get, setf=setf):
                    old = get()
                    setf(int(n))
                    return old
                return ctl
    except Exception:
        return None
    return None


def cpu_baseline(name, scale, P, applies, matvecs, samples=1):
    cs = _CpuSampler(name, scale, P)
    res = [cs.sample(applies, matvecs) for _ in range(samples)]
    v = float(np.mean([r["value"] for r in res]))
    out = {"value": v, "unit": "s", "cores": cs.threads, "kind": "port",
           "sample": cs.describe(applies, matvecs), "samples": res}
    full = _full_run(name, P, scale)
    if full:
        out["full_run_measured"] = full
    return out


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    P = args.P if args.P is not None else DEFAULT_P.get(args.config)
    full = _full_run(args.config, P, args.scale)
    # the solve's counts: the oracle's own full run when it was measured, else the GPU's
    applies = full["precond_applications"] if full else 312
    matvecs = applies + 2
    cs = _CpuSampler(args.config, args.scale, P)
    # one step = one measured wave (~25 s of CPU work for c3 P=64 on 16 cores); at most
    # 1 warm-up and 3 timed waves so that the arm finishes within a few minutes whatever K
    n_warm, n_steps = min(args.warmup, 1), max(1, min(args.steps, 3))
    for _ in range(n_warm):
        cs.sample(applies, matvecs)
    vals = []
    t0 = time.perf_counter()
    for _ in range(n_steps):
        vals.append(cs.sample(applies, matvecs)["value"])
    wall = time.perf_counter() - t0
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "preconditioned solve time-to-tolerance (s)", "value": v,
        "unit": "s", "n_gpus": ws, "steps": n_steps, "warmup": n_warm,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1e3 * wall / n_steps, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload(args.config, P, args.scale), "scale": args.scale},
        "cpu_baseline": {"kind": "port", "cores": cs.threads,
                         "sample": cs.describe(applies, matvecs), "value": v, "unit": "s"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if full:
        line["cpu_baseline"]["full_run_measured"] = full
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def run_ours(args):
    import torch

    from paper_2504_11167_b200 import api, configs

    ws, rank, local = _dist()
    comm = None
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # a dedicated stream shared by torch and the library: the CUDA events of the timed
    # region are recorded on the stream every kernel of the step is launched on
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx = api.Context(local, stream.cuda_stream)
    if ws > 1:
        # the in-library NCCL data plane: exchanges enqueued on the context stream
        from paper_2504_11167_b200.dist import LibNcclComm

        comm = LibNcclComm(ctx)
    assert ctx.stream == stream.cuda_stream != 0
    P = args.P if args.P is not None else DEFAULT_P.get(args.config)
    cfg = configs.make_config(args.config, args.scale, P)
    # c5: the 8 FEAST contour systems are independent -- replicas, rank q solves shift q % 8
    shift = rank % 8 if args.config == "c5" else None
    matrix = cfg.system(shift) if shift is not None else cfg.matrix
    rhs_h = np.asfortranarray(cfg.rhs.astype(np.complex128) if shift is not None else cfg.rhs)
    A = api.CsrMatrix.from_csr(ctx, matrix)
    scfg = api.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=3000)
    b_dev = torch.from_numpy(rhs_h).cuda()
    x_dev = torch.empty_like(b_dev)
    dmma_peak = ctx.dmma_peak_tflops()
    i8_peak = ctx.i8_peak_tops()

    def make_fact(Amat):
        if comm is None:
            return api.factorize(ctx, Amat, scfg)
        from paper_2504_11167_b200.dist import DistFactorization

        return DistFactorization(ctx, Amat, scfg, comm)

    def step():
        F = make_fact(A)
        x, rep, _ = api.solve(A, b_dev, it=it, F=F, x_out=x_dev)
        return F, rep

    for _ in range(args.warmup):
        F, rep = step()
        del F
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    # CUDA events only around the launches the rooflines need (the bulk LU update, the
    # apply's sweeps, interface and recovery): an event pair around every one of the ~7000
    # launches of a step costs ~10 ms; the all-class breakdown comes from one extra
    # untimed step below
    ctx.set_profiling(True, classes=("lu_update", "band_solve", "iface_apply", "recovery"))
    ctx.kernel_times(reset=True)
    l0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, infos = [], []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            F, rep = step()
            reps.append(rep)
            infos.append(F.info)
            del F
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - l0
    kt = ctx.kernel_times(reset=True)
    ctx.set_profiling(True)
    F, rep_b = step()  # untimed: the per-class breakdown of one step
    del F
    torch.cuda.synchronize()
    kt_all = ctx.kernel_times(reset=True)
    ctx.set_profiling(False)
    # the same LU with the DMMA trailing update (LRS_LU_I8=0), untimed, for the bench line
    t_lu_dmma = None
    if comm is None:
        old = os.environ.get("LRS_LU_I8")
        os.environ["LRS_LU_I8"] = "0"
        try:
            Fd = api.factorize(ctx, A, scfg)
            t_lu_dmma = Fd.info["t_lu"]
            del Fd
        finally:
            if old is None:
                os.environ.pop("LRS_LU_I8")
            else:
                os.environ["LRS_LU_I8"] = old
    ms = ev0.elapsed_time(ev1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = ms / 1e3

    # ---- e2e: public C-ABI with host buffers (CSR upload + factorize + solve + x back)
    e2e_vals = []
    csr = matrix
    h2d = 8 * (csr.n + 1) + 8 * csr.nnz + csr.values.nbytes + rhs_h.nbytes
    d2h = rhs_h.nbytes

    def pinned(a):  # a page-locked host copy (numpy view), made outside the timed region
        t = torch.empty(a.size, dtype=torch.from_numpy(a[:0].copy()).dtype, pin_memory=True)
        v = t.numpy()
        v[:] = np.ravel(a, order="F")
        return v, t
    (h_rp, _k1), (h_ci, _k2), (h_va, _k3) = (pinned(csr.row_ptr), pinned(csr.col_idx),
                                             pinned(csr.values))
    h_b, _k4 = pinned(rhs_h)
    h_b = h_b.reshape(rhs_h.shape, order="F")
    # e2e: 1 warm-up + min(steps, 5) timed (each c3 step re-uploads 300 MB of CSR and
    # refactorizes 87 GB of band factors; five steps bound the run time)
    e2e_warm, e2e_steps = 1, min(args.steps, 5)
    for i in range(e2e_warm + e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A2 = api.CsrMatrix(ctx, csr.n, h_rp, h_ci, h_va)
        F2 = make_fact(A2)
        xh, rep2, F2 = api.solve(A2, h_b, it=it, F=F2)
        dt = time.perf_counter() - t0
        del F2, A2
        if i >= e2e_warm:
            e2e_vals.append(dt)
    e2e = float(np.mean(e2e_vals))
    if ws > 1:
        t = torch.tensor([e2e], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())

    # ---- roofline: dominant kernel = band-LU trailing update (DMMA, FP64 tensor core)
    info = infos[-1]
    upd_ms, upd_n = kt["lu_update"]
    # algorithmic (no-fill) flops of the bulk trailing update: for pivot column j (row tile
    # K = j / 128) the rank-1 update of rows and columns beyond the look-ahead row/column
    # (>= K + 2; >= K0 + 3 for the two-step launches of steps K0, K0 + 1); the look-ahead
    # rows/columns are critical-path work timed with the panel
    lu_steps = int(info.get("lu_pairs", 0))
    lu_upd_flops = sum(_rest_update_flops(s, info["kl"], info["ku"], info["nb"], lu_steps)
                       for s in _partition_sizes(cfg.matrix.n, cfg.P))
    # the symmetric schedule (info.lu_sym) forms the lower trailing tiles only: its FP64-
    # equivalent work is the full update's scaled by the share of tiles it computes
    sym_scale = 1.0
    if info.get("lu_sym") and lu_steps:
        sizes = _partition_sizes(cfg.matrix.n, cfg.P)
        full = sum(_i8_bulk_tiles(s, info["wl"], info["wu"], info["nb"], lu_steps) for s in sizes)
        half = sum(_i8_bulk_tiles(s, info["wl"], info["wu"], info["nb"], lu_steps, True)
                   for s in sizes)
        sym_scale = half / full if full else 1.0
    lu_upd_flops *= sym_scale
    per_launch_flops = lu_upd_flops * args.steps / max(upd_n, 1)
    avg_launch_s = upd_ms / max(upd_n, 1) / 1e3
    achieved_tf = per_launch_flops / avg_launch_s / 1e12 if upd_n else 0.0
    # apply (HBM): band_solve launches of the Krylov phase
    solve_ms, solve_n = kt["band_solve"]
    napply = sum(r.precond_applications for r in reps)
    apply_bytes = info["apply_bytes"]
    peaks, peak_src = _peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # D-stage: 2 band_solve launches per apply (L, U) + the spike-construction solves
    apply_ms_each = None
    if napply:
        apply_ms_each = (kt["band_solve"][0] + kt["iface_apply"][0] + kt["recovery"][0]) / 1.0
    total_ms = sum(v[0] for v in kt_all.values())
    if info.get("lu_int8"):
        # INT8 ops the launch issues: 28 digit-slice products (M = N = 128, K = 128 x steps)
        # per 128 x 128 tile of the bulk update
        tiles = sum(_i8_bulk_tiles(s, info["wl"], info["wu"], info["nb"], lu_steps,
                                   bool(info.get("lu_sym")))
                    for s in _partition_sizes(cfg.matrix.n, cfg.P))
        ops_launch = (tiles * args.steps * 2.0 * 128 * 128 * 128 * lu_steps * I8_PRODUCTS /
                      max(upd_n, 1))
        achieved_tops = ops_launch / avg_launch_s / 1e12 if upd_n else 0.0
        roofline = {"bound": "tensor",
                    "kernel": f"lu_i8_gemm_kernel<4, {lu_steps}> (INT8-sliced FP64 {lu_steps}-step "
                              "trailing update, tcgen05.mma kind::i8)",
                    "achieved": achieved_tops, "peak": i8_peak, "unit": "TOPS (int8)",
                    "frac": achieved_tops / i8_peak if i8_peak else None,
                    "peak_source": "in-run INT8 tcgen05 microbenchmark (M=128, N=256, resident "
                                   "operands); nominal dense 4.5 POPS",
                    # DRAM read + write of one (large, K = 20) launch from `ncu --set full`
                    # (profiles/r02_ncu_summaries.txt): the C tiles' read-modify-write
                    "traffic": _ncu_traffic(f"{args.config}_P{cfg.P}_lu_i8").get("value"),
                    "traffic_source": _ncu_traffic(f"{args.config}_P{cfg.P}_lu_i8").get("source"),
                    "launches": int(upd_n), "avg_launch_ms": avg_launch_s * 1e3,
                    "int8_ops_per_launch": ops_launch,
                    # 1.0: every trailing tile; ~0.51: the symmetric schedule's lower tiles
                    # (the ops counted above are the ones issued, not the full schedule's)
                    "tiles_share_of_full_schedule": sym_scale,
                    "fp64_equiv": {"achieved": achieved_tf, "unit": "TFLOP/s",
                                   "dmma_peak": dmma_peak,
                                   "ratio_to_dmma_peak": achieved_tf / dmma_peak if dmma_peak else None,
                                   "flops_per_launch": per_launch_flops}}
    else:
        roofline = {"bound": "tensor",
                    "kernel": ("lu_gemm_kernel<4> (two-step DMMA trailing update)"
                               if info.get("lu_pairs") else "lu_gemm_kernel<1> (DMMA trailing update)"),
                    "achieved": achieved_tf, "peak": dmma_peak, "unit": "TFLOP/s",
                    "frac": achieved_tf / dmma_peak if dmma_peak else None,
                    "peak_source": "in-run FP64 DMMA microbenchmark (MEASURED_PEAKS.json has no FP64); "
                                   "nominal 148 SM x 64 FMA x 2 x 1.965 GHz = 37.2",
                    "traffic": None, "launches": int(upd_n), "avg_launch_ms": avg_launch_s * 1e3,
                    "flops_per_launch": per_launch_flops}
    apply_rl = _apply_roofline(kt, reps, info, hbm_peak, peak_src, args.steps,
                               f"{args.config}_P{cfg.P}_apply")
    upd_ms_step = upd_ms / max(args.steps, 1)
    roofline["ms_per_step"] = upd_ms_step
    dominant = roofline
    if apply_rl and apply_rl["ms_per_step"] > upd_ms_step:
        dominant = apply_rl
    line = {
        "metric": "preconditioned solve time-to-tolerance (s)",
        "value": value, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False,
        "scaling": "weak" if shift is not None else "strong",
        "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload(args.config, P, args.scale),
                   "scale": args.scale, "P": cfg.P,
                   "parallelism": (f"partition-sharded: {cfg.P} partitions over {ws} GPUs (NCCL)"
                                   if ws > 1 else "1 GPU, all partitions"),
                   "l2": (f"inputs larger than L2 ({info['apply_bytes'] / 1e9:.0f} GB of band "
                          "factors streamed per apply)")},
        "iterations": reps[-1].iterations, "precond_applications": reps[-1].precond_applications,
        "residual_final": reps[-1].residual_final,
        "t_factorize_s": info["t_factorize"], "t_lu_s": info["t_lu"], "t_spikes_s": info["t_spikes"],
        "t_solve_s": reps[-1].wall_time,
        # host round trips of the solve: transport calls, stream syncs forced before them
        # (0: the in-library NCCL plane is stream-ordered), syncs to read Krylov scalars
        "round_trips": reps[-1].round_trips,
        # the band LU's bulk update ran INT8-sliced on tcgen05 (lu_int8 = 1) or DMMA;
        # t_lu_dmma_s = the same LU with LRS_LU_I8=0 (one extra untimed factorization)
        "lu_int8": int(info.get("lu_int8", 0)), "lu_sym": int(info.get("lu_sym", 0)),
        "t_lu_dmma_s": t_lu_dmma,
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        # the dominant kernel of the step (by CUDA-event time per step) carries `roofline`;
        # the other one is reported beside it
        "roofline": dominant,
        # FP64-equivalent rate of the whole LU on the flops it forms (the no-fill gbtrf count,
        # scaled by the symmetric schedule's tile share when lu_sym = 1)
        "roofline_lu_all": {"achieved": sym_scale * info["lu_flops"] / info["t_lu"] / 1e12,
                            "unit": "TFLOP/s", "work_share_of_gbtrf": sym_scale,
                            "frac": sym_scale * info["lu_flops"] / info["t_lu"] / 1e12 / dmma_peak},
        "roofline_apply": apply_rl,
        "roofline_lu_update": roofline,
        # per-class CUDA-event breakdown of one extra (untimed, fully profiled) step
        "kernel_ms_per_step": {k: v[0] for k, v in kt_all.items()},
        "kernel_launches_per_step": {k: v[1] for k, v in kt_all.items()},
        "kernel_ms_total_share": {k: (v[0] / total_ms if total_ms else 0) for k, v in kt_all.items()},
    }
    clocks = clk.summary()
    line["clocks"] = clocks
    if shift is not None:
        line["config"]["shift"] = {"index": shift, "z": [cfg.shifts[shift].real, cfg.shifts[shift].imag],
                                   "n_rhs": int(rhs_h.shape[1])}
        line["dtype"] = "c128"
    if rank == 0 and not args.no_cpu_baseline and shift is None:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, args.scale, P,
                                                reps[-1].precond_applications, reps[-1].matvecs)
        except Exception as e:  # baseline failure must not hide the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    del apply_ms_each, solve_ms, solve_n, napply, apply_bytes
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def _rest_update_flops(s, kl, ku, nb=128, steps=0):
    j = np.arange(s, dtype=np.int64)
    K = j // nb
    # single steps: rows/cols >= K + 2; D-step launches (D = 2: rank 256, D = 4: rank 512) for
    # steps K0 .. K0+D-1, K0 = K - K % D: rows/cols >= K0 + 2D (look-ahead depth D)
    lo = ((K - K % steps + 2 * steps) if steps else K + 2) * nb
    ni = np.clip(np.minimum(j + kl, s - 1) - np.maximum(j + 1, lo) + 1, 0, None).astype(np.float64)
    nc = np.clip(np.minimum(j + ku, s - 1) - np.maximum(j + 1, lo) + 1, 0, None).astype(np.float64)
    return float(2.0 * np.sum(ni * nc))


def _i8_bulk_tiles(s, wl, wu, nb=128, steps=2, sym=False):
    """128 x 128 tiles of the INT8 bulk launches (I, J >= K + 2D of each D-step update; the
    symmetric schedule forms the lower triangle I >= J of that window only)."""
    T = -(-s // nb)
    tot = 0
    for K in range(0, T, steps):
        ni = max(0, min(K + steps - 1 + wl, T - 1) - (K + 2 * steps) + 1)
        nj = max(0, min(K + steps - 1 + wu, T - 1) - (K + 2 * steps) + 1)
        tot += ni * (ni + 1) // 2 if sym else ni * nj
    return tot


def _partition_sizes(n, P):
    return [n // P + (1 if i < n % P else 0) for i in range(P)]


def _ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch (or per apply) of one
    `ncu --set full` capture, committed in profiles/ncu_traffic.json by scripts/ncu_summary.py."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(key, {})
    except (OSError, ValueError):
        return {}


def _apply_roofline(kt, reps, info, hbm_peak, peak_src, steps, cfg_key):
    """Per-apply achieved GB/s of the D-stage (2 band_solve launches) + iface + recovery
    in the Krylov phase.  band_solve launches of the spike setup (2l columns, multi-RHS)
    are a different shape, so the per-launch average here is restricted by count."""
    applies = sum(r.precond_applications for r in reps)
    ms, n = kt["band_solve"]
    if not applies or not n:
        return None
    # the Krylov-phase sweeps: one fused L + U launch per apply (band_solve_lu1_kernel), or
    # two launches with LRS_SOLVE_FUSED=0
    per_apply_launches = 1 if n <= applies else 2
    ms_iface = kt["iface_apply"][0] + kt["recovery"][0]
    sweeps_ms = ms * (per_apply_launches * applies / n)
    per_apply_ms = (sweeps_ms + ms_iface) / applies
    gbs = info["apply_bytes"] / (per_apply_ms / 1e3) / 1e9
    traffic = _ncu_traffic(cfg_key)
    return {"bound": "hbm",
            "kernel": "band_solve_lu1_kernel (the one-RHS L and U dataflow sweeps of the "
                      "apply, one launch) + iface + recovery",
            "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
            # DRAM read + write of one apply's two sweeps from `ncu --set full`
            # (profiles/r02_ncu_summaries.txt): 2.6% above the algorithmic bytes
            "traffic": traffic.get("value"), "traffic_source": traffic.get("source"),
            "bytes_per_apply": info["apply_bytes"], "ms_per_apply": per_apply_ms,
            # the two sweeps alone (the iface / recovery kernels and launch gaps excluded)
            "sweeps_gbs": info["apply_bytes"] / (sweeps_ms / applies / 1e3) / 1e9,
            "ms_per_step": per_apply_ms * applies / steps,
            "frac_of_8TBs_nominal": gbs / 8000.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--P", type=int, default=None, help="partitions (default: c3 64, c2 8)")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
