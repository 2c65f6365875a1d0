#!/usr/bin/env python
"""Benchmark of the MU-NMF hot path (BASELINE.json metric: MU iters/sec and A-pass GB/s vs the
HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload dense|sparse|ooc]

A "step" is one MU iteration (W update then H update; error every 10 iterations as the
reference default). Default workload = config 2: synthetic dense 65536 x 65536 f32 A, k = 32,
row-partitioned over N GPUs (strong scaling), one JSON line on rank 0; at N > 1 the line also
carries a "weak" sub-record (65536 rows per GPU, m = N x 65536: the north star's weak-scaling
target) and --scaling weak makes that the main measurement.
  --workload sparse : config 3, CSR 2^22 x 2^22, density 1e-5 (reference generator), k = 32
  --workload ooc    : config 4 (scaled to this host's RAM): A in pinned host memory, streamed
                      over the host link every iteration, k = 64

--impl reference times the reference's own CPU solver (oracle/_ref, compiled from the
/root/reference sources; the oracle port if absent) on this box's host cores, one MU
iteration per step on a bounded row sample, extrapolated to the full matrix.
"""
import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CPU_CORES = os.cpu_count() or 1
os.environ.setdefault("OMP_NUM_THREADS", str(CPU_CORES))

# stdout carries exactly the one JSON line: native libraries (NCCL's version banner, ...) write
# to file descriptor 1 directly, so fd 1 is pointed at stderr and the line goes to a saved copy
_JSON_FD = None


def emit(obj):
    global _JSON_FD
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)


def _quiet_stdout():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["dense", "sparse", "ooc", "select"], default="dense")
    # (--rows / --cols aliases: torchrun's own parser swallows an abbreviated --m)
    p.add_argument("--m", "--rows", dest="m", type=int, default=None)
    p.add_argument("--n", "--cols", dest="n", type=int, default=None)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--density", type=float, default=1e-5)
    p.add_argument("--ooc-gb", type=float, default=64.0, help="host A slab per rank (GB) for --workload ooc")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-e2e-f64", action="store_true", help="skip the reference-shaped f64 pageable e2e run")
    p.add_argument("--no-sparse", action="store_true", help="dense workload: skip the config-3 sub-record")
    p.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                   help="strong (default): the same m at every N (value = whole-job it/s, ideally N x); "
                        "weak: m = N x --m rows (a fixed slab per GPU)")
    p.add_argument("--no-weak", action="store_true",
                   help="N > 1, strong: skip the weak-scaling sub-record of the dense line")
    p.add_argument("--ref-sample", action="store_true",
                   help="--impl reference: time a 1024-row sample instead of the full workload")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    # --workload select (config 5: select_k over k=2..16 on dense 32768 x 16384)
    p.add_argument("--k-min", type=int, default=2)
    p.add_argument("--k-max", type=int, default=16)
    p.add_argument("--perturbations", type=int, default=16)
    p.add_argument("--select-iters", type=int, default=500, help="max_iters per run (reference CLI default 500)")
    a = p.parse_args()
    dflt = {"dense": (65536, 65536, 32), "sparse": (1 << 22, 1 << 22, 32), "ooc": (None, 65536, 64),
            "select": (32768, 16384, 9)}[a.workload]
    a.m = a.m or dflt[0]
    a.n = a.n or dflt[1]
    a.k = a.k or dflt[2]
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Clock / throttle sampling during the timed region (B200_PROFILING.md clocks line).

    NVML is polled in-process every ~2 ms from a thread (ctypes releases the GIL while the solve
    runs), so even a ~70 ms timed region (config 2 at N=4) gets samples; only samples taken
    after ``__enter__`` returns count. Falls back to ``nvidia-smi -lms 100`` without pynvml."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason{HwSlowdown,HwThermalSlowdown,SwThermalSlowdown,SwPowerCap}

    def __init__(self, index):
        self.index = str(index)
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (t, sm_mhz, max_mhz, power_w, reasons bitmask)
        self.stop = threading.Event()
        self.t_begin = None

    def _nvml_handle(self, pynvml):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").strip()
        ent = [x.strip() for x in vis.split(",") if x.strip()] if vis else []
        local = int(self.index)
        if ent and local < len(ent):
            e = ent[local]
            if e.isdigit():
                return pynvml.nvmlDeviceGetHandleByIndex(int(e))
            return pynvml.nvmlDeviceGetHandleByUUID(e)
        return pynvml.nvmlDeviceGetHandleByIndex(local)

    def _poll(self, pynvml, h):
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1e3
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((time.perf_counter(), float(sm), float(mx), pw, int(rs)))
            except Exception:
                pass
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = self._nvml_handle(pynvml)
            self.nvml = pynvml
            self.t = threading.Thread(target=self._poll, args=(pynvml, h), daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                              "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except Exception:
                self.proc = None
        self.t_begin = time.perf_counter()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=5)
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, pw, reasons = [], [], [], set()
        for t, s, m, p, rs in self.samples:
            if t < self.t_begin:
                continue
            sm.append(s), mx.append(m), pw.append(p)
            for nm, bit in zip(self.NAMES, self.BITS):
                if rs & bit:
                    reasons.add(nm)
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9 or f[0] != self.index:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None,
                "source": "nvml" if self.samples else "nvidia-smi"}


# ----------------------------------------------------------------------------- CPU reference
def _ref_impl():
    import oracle

    impl = oracle.ref if oracle.ref.available else oracle.port
    return impl, ("reference" if impl is oracle.ref else "port")


def cpu_reference_dense(m, n, k, seconds, steps=None, warmup=0):
    """Reference CPU solver, one MU iteration per step on a 1024-row sample of the uniform A;
    returns (it/s extrapolated to m rows, cpu_baseline dict). Cost is linear in rows here
    (every term of the iteration is O(rows * n * k) except O(n k^2) ones, < 0.1%)."""
    import numpy as np

    import oracle

    impl, kind = _ref_impl()
    rows = 1024
    a = impl.uniform_dense(rows, n, 42, 99)
    w, h = oracle.port.init_factors(m, n, k, 0)
    w = np.ascontiguousarray(w[:rows])
    if kind == "reference":
        hnd = impl.dense_handle(a)

        def step():
            impl.mu_iteration_handle(hnd, w, h)
    else:
        def step():
            impl.mu_iteration(a, w, h)
    for _ in range(max(1, warmup)):
        step()
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and (time.perf_counter() > t_end or len(times) >= 50):
            break
    if kind == "reference":
        impl.dense_free(hnd)
    per_it = sum(times) / len(times)
    rate = (1.0 / per_it) * rows / m
    return rate, {"value": rate, "unit": "it/s", "cores": int(os.environ.get("OMP_NUM_THREADS", CPU_CORES)),
                  "kind": kind,
                  "sample": f"{len(times)} MU iterations (W then H update, f64) on a {rows} x {n} row sample of the "
                            f"uniform A, k={k}; {per_it:.3f} s/iter scaled by {rows}/{m} rows (cost is linear in rows)"}


def cpu_reference_sparse(samples, m, k, seconds):
    """samples: [(rows_i, CsrMatrix)] row samples of the same matrix. The reference's CSR
    iteration costs a + b*rows (a = the O(n k^2) H-side terms); fit a, b from two sample
    sizes and extrapolate to m rows."""
    import numpy as np

    import oracle

    impl = oracle.ref
    if not impl.available:
        return None, None
    kind = "reference"
    pts = []
    for rows, s in samples:
        n = s.cols
        w0, h0 = oracle.port.init_factors(rows, n, k, 0)
        hnd = impl.csr_handle(s.row_ptr, s.col_idx, s.values, rows, n)
        per = []
        t_end = time.perf_counter() + seconds / len(samples)
        try:
            while True:
                t0 = time.perf_counter()
                impl.mu_iteration_csr_handle(hnd, w0, h0)  # loop body of nmf_serial, no error check
                per.append(time.perf_counter() - t0)
                if time.perf_counter() > t_end or len(per) >= 5:
                    break
        finally:
            impl.csr_free(hnd)
        pts.append((rows, min(per), s.nnz))
    (r1, t1, _), (r2, t2, _) = pts[0], pts[-1]
    # the fixed O(n k^2) part dominates small samples; a noisy slope is clamped at 0, which can
    # only flatter the reference (per_full >= the larger sample's own time)
    b = max((t2 - t1) / (r2 - r1), 0.0)
    a = t1 - b * r1
    per_full = max(a + b * m, t2)
    rate = 1.0 / per_full
    return rate, {"value": rate, "unit": "it/s", "cores": int(os.environ.get("OMP_NUM_THREADS", CPU_CORES)),
                  "kind": kind,
                  "sample": f"reference MU iteration (nmf_serial loop body, no error check) on row samples "
                            f"{[(p[0], p[2]) for p in pts]} (rows, nnz) of the same CSR; fit t = a + b*rows "
                            f"(a={a:.3f}s, b={b:.3e}s/row) extrapolated to {m} rows: {per_full:.1f} s/iter"}


# ----------------------------------------------------------------------------- helpers
FUSED = "mu_fused (A.H^T, W update, A^T.W; A read from HBM once)"


def roofline(info, bytes_per_launch, peak, peak_src, traffic=None, bound="hbm", unit="GB/s"):
    per = {}
    for name, key in (("aht_pass (A.H^T)", "aht_pass_ms"), ("wta_pass (A^T.W)", "wta_pass_ms"),
                      (FUSED, "fused_pass_ms")):
        launches = int(info.get(key.replace("_ms", "_launches"), 0))
        if launches:
            per[name] = info[key] / launches
    dom = max(per, key=per.get)
    b = bytes_per_launch[dom] if isinstance(bytes_per_launch, dict) else bytes_per_launch
    achieved = b / (per[dom] * 1e-3) / 1e9
    tr = traffic.get(dom.split()[0]) if traffic else None
    out = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
           "traffic": tr, "kernel": dom, "algorithmic_bytes_per_launch": b, "avg_launch_ms": per[dom],
           "per_kernel_ms": per, "peak_source": peak_src}
    if dom == FUSED:
        # both A passes of the iteration in one launch: the algorithmic bytes (2 |A| + factors,
        # SURVEY.md §8(d)) exceed what crosses HBM (A once + the re-reads that missed L2), so frac
        # can pass 1; frac_dram is the DRAM bytes actually moved (ncu) over the same time
        out["note"] = ("one-pass kernel: A.H^T, the W update and A^T.W in one launch; algorithmic bytes = both A "
                       "passes (2|A| + factors), the second served from L2")
        if tr:
            out["frac_dram"] = tr / (per[dom] * 1e-3) / 1e9 / peak
    return out


def bench_select(args, nmf, np, torch, ctx, comm, rank, world, local, barrier, max_over_ranks):
    """Config 5: one select_k sweep (k_min..k_max, P perturbations, max_iters per run) on a dense
    m x n A resident on every rank (replicas; the P runs of each k spread over the ranks).
    value = MU iterations executed by the sweep (all runs, all ranks) / sweep time (CUDA events
    on the caller's stream around the synchronous call, max over ranks; includes the GPU
    perturbations, the host clustering / silhouette and the per-k W exchange)."""
    m, n = args.m, args.n
    K = args.steps
    hbm, peak_src = peaks()
    ctx.set_problem(m, n, args.k_min, 0, m)
    ctx.generate_dense_uniform(42, 99)
    host = np.empty((m, n), np.float32)
    ctx.download_dense(host)
    cfg = nmf.SelectionConfig(k_min=args.k_min, k_max=args.k_max, n_perturbations=args.perturbations,
                              delta=0.03, sil_threshold=0.75, seed=0,
                              nmf=nmf.NmfConfig(max_iters=args.select_iters, error_check_interval=10, eta=1e-6,
                                                device=local))
    from paper_2202_09518_b200.nmf import _select_on

    # warm-up: a 2-run sweep at k_min with a few iterations (kernels, graphs, clustering code)
    wcfg = nmf.SelectionConfig(k_min=args.k_min, k_max=args.k_min, n_perturbations=2, seed=1,
                               nmf=nmf.NmfConfig(max_iters=max(3, args.warmup), error_check_interval=10, eta=0.0,
                                                 device=local))
    _select_on(ctx, m, wcfg)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        rep = _select_on(ctx, m, cfg)
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    sweep_s = max_over_ranks(ev0.elapsed_time(ev1)) / 1e3
    iters = sum(r.iterations for r in rep.records)
    value = iters / sweep_s
    # e2e: the public call on host memory = the A upload (pinned H2D, timed) + the sweep
    nmf.check(nmf._capi.lib().oocnmf_host_register(host.ctypes.data, host.nbytes))
    try:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.set_problem(m, n, args.k_min, 0, m)
        ctx.load_dense(host)
        e1.record()
        torch.cuda.synchronize()
        upload_s = max_over_ranks(e0.elapsed_time(e1)) / 1e3
    finally:
        nmf._capi.lib().oocnmf_host_unregister(host.ctypes.data)
    achieved = 2 * m * n * 4 * iters / world / sweep_s / 1e9  # A bytes streamed per GPU per second
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kmid = (args.k_min + args.k_max) // 2
        _, cpu = cpu_reference_dense(m, n, kmid, args.cpu_seconds)
        cpu["sample"] += f" (k = {kmid}, the middle of the sweep)"
    if rank == 0:
        out = {"metric": f"MU iters/sec across a select_k sweep (dense {m}x{n}, k={args.k_min}..{args.k_max}, "
                         f"P={args.perturbations})",
               "value": value, "unit": "it/s", "n_gpus": world, "steps": iters, "warmup": 1,
               "ms_per_step": sweep_s * 1e3 / iters, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f32", "data": "synthetic",
               "config": {"workload": f"model selection (config 5): select_k k={args.k_min}..{args.k_max}, "
                                      f"P={args.perturbations}, delta 0.03, max_iters {args.select_iters}, eta 1e-6 "
                                      f"on dense synthetic {m}x{n} uniform A (CounterRng(42,99)), runs spread "
                                      f"over {world} rank(s) as replicas",
                          "m": m, "n": n, "k_min": args.k_min, "k_max": args.k_max,
                          "perturbations": args.perturbations, "parallelism": f"replicas-x{world}",
                          "l2": "A (2.1 GB) >> 126 MB L2 (no flush needed)"},
               "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                            "frac": achieved / hbm, "traffic": None,
                            "kernel": "whole sweep: two A passes per MU iteration, amortised over perturbation, "
                                      "factor updates, error checks and host clustering",
                            "peak_source": peak_src},
               "cpu_baseline": cpu,
               "e2e": {"value": iters / (sweep_s + upload_s), "unit": "it/s",
                       "h2d_bytes_per_step": m * n * 4 / iters,
                       "d2h_bytes_per_step": sum(m * r.k * 8 * (args.perturbations + 1) for r in rep.records) / iters,
                       "note": f"A uploaded from pinned host memory ({upload_s:.3f} s, timed) + the sweep; W factors "
                               f"and medians come back to the host for clustering"},
               "clocks": clk.summary(), "sweep_s": sweep_s, "chosen_k": rep.chosen_k,
               "records": [[r.k, r.runs_used, round(r.min_silhouette, 4), round(r.mean_relative_error, 6),
                            r.iterations] for r in rep.records]}
        emit(out)
    if comm:
        comm.close()


def reference_arm(args, rank, K, W, k, world=1):
    """--impl reference: the reference's own CPU solver (oracle/_ref) on this box's host cores.

    dense (default): the SAME configuration as our arm — the full 65536 x 65536 A (f64, the
    reference's type, values rounded from the same f32 uniform draw), W warm-up MU iterations,
    then one timed nmf_serial of K iterations with the reference's check cadence (every 10 and
    the last; src/nmf_serial.cpp:83-117), so value = K / that time. When the host cannot hold the
    f64 A (or --ref-sample is given) it falls back to the row-sample extrapolation."""
    if rank != 0:
        return
    if world > 1 and os.environ.get("OMP_NUM_THREADS") == "1":
        # torchrun pins OMP_NUM_THREADS=1 per process; rank 0 alone runs the reference here, with
        # every host core as at N = 1 (set before the OpenMP runtime of oracle/_ref loads)
        os.environ["OMP_NUM_THREADS"] = str(CPU_CORES)
    m, n = (args.m or 65536) * (world if args.scaling == "weak" else 1), args.n
    if args.workload != "dense":
        emit({"impl": "reference", "unavailable": "--impl reference implemented for the default (dense) workload only"})
        return
    workload = f"dense synthetic {m}x{n} f32 uniform A (CounterRng(42,99)), k={k}, RNMF row slabs"
    metric = f"MU iters/sec (dense {m}x{n}, k={k}, 1D row-partitioned, NCCL all-reduce)"
    import numpy as np

    impl, kind = _ref_impl()
    cores = int(os.environ.get("OMP_NUM_THREADS", CPU_CORES))
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES")
    except (ValueError, OSError):
        ram = 0
    # the full same-config run at N = 1 (the headline ratio); under torchrun (N > 1, where weak
    # scaling makes A N times larger) the bounded row-sample fit keeps the arm within minutes
    full = not args.ref_sample and world == 1 and kind == "reference" and m * n * 8 < 0.8 * ram
    if full:
        import oracle

        t0 = time.perf_counter()
        hnd = impl.dense_uniform_handle(m, n, 42, 99, round_f32=True)  # built in place, OpenMP
        gen_s = time.perf_counter() - t0
        w, h = oracle.port.init_factors(m, n, k, 0)
        try:
            # one warm-up MU iteration is enough for a CPU solver (pages touched, threads up);
            # each costs ~13 s at this size
            w_cpu = min(W, 1)
            t0 = time.perf_counter()
            for _ in range(w_cpu):
                impl.mu_iteration_handle(hnd, w, h)  # the loop body of nmf_serial (nmf_serial.cpp:84-101)
            warm_s = time.perf_counter() - t0
            # bound the arm's wall time (OOCNMF_REF_BUDGET_S, default 360 s for generation,
            # warm-up and the timed solve) so the run ends within minutes for any --steps: the
            # rate is per iteration of the same full-size solve, so timing fewer of them measures it
            budget = float(os.environ.get("OOCNMF_REF_BUDGET_S", 360))
            per_it = 1.25 * warm_s / max(w_cpu, 1)  # (+ the error checks the warm-up step skips)
            k_run = K if per_it <= 0 else max(10, min(K, int((budget - gen_s - warm_s) / per_it)))
            t0 = time.perf_counter()
            r = impl.nmf_serial_handle(hnd, m, n, k, max_iters=k_run, interval=10, eta=0.0, seed=0)
            secs = time.perf_counter() - t0
        finally:
            impl.dense_free(hnd)
        rate = k_run / secs
        cb = {"value": rate, "unit": "it/s", "cores": cores, "kind": kind,
              "sample": f"the full workload: nmf_serial (f64) on the {m}x{n} A, k={k}, {k_run} iterations"
                        f"{'' if k_run == K else f' (of the requested {K}: wall-time budget)'} with error "
                        f"checks every 10 and on the last ({len(r.trace_err)} checks, final error "
                        f"{r.trace_err[-1]:.6f}), after {w_cpu} warm-up MU iteration(s) ({warm_s:.1f} s); A generated in "
                        f"{gen_s:.1f} s (not timed)",
              "same_config": True}
        extra = {"timed_s": secs, "timed_iterations": k_run, "final_rel_error": float(r.trace_err[-1])}
    else:
        rate, cb = cpu_reference_dense(m, n, k, args.cpu_seconds, steps=K, warmup=W)
        cb["sample"] = cb["sample"].replace("MU iterations", f"timed MU iterations after {W} warm-up")
        cb["same_config"] = False
        extra = {}
    out = {"impl": "reference", "metric": metric, "value": rate, "unit": "it/s", "n_gpus": args.gpus,
           "steps": K, "warmup": W, "ms_per_step": 1e3 / rate, "higher_is_better": True,
           "scaling": "weak" if args.scaling == "weak" else "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": workload, "m": m, "n": n, "k": k, "parallelism": f"host cores ({cores} threads)",
                      "error_check_interval": 10},
           "cpu_baseline": cb,
           "e2e": {"value": rate, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    out.update(extra)
    emit(out)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    K, W, k = args.steps, max(3, args.warmup), args.k

    if args.impl == "reference":
        return reference_arm(args, rank, K, W, k, world)

    import numpy as np
    import torch

    import paper_2202_09518_b200 as nmf

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t)
        return float(t.item())

    comm = nmf.DistComm(rank, world, local) if world > 1 else None
    ctx = comm.ctx if comm else nmf.Context(local)
    if args.workload == "select":
        return bench_select(args, nmf, np, torch, ctx, comm, rank, world, local, barrier, max_over_ranks)
    env = dict(nmf=nmf, np=np, torch=torch, ctx=ctx, rank=rank, world=world, local=local, barrier=barrier,
               max_over_ranks=max_over_ranks, sum_over_ranks=sum_over_ranks)
    out = run_workload(args, args.workload, args.m, args.n, k, K, W, env)
    if args.workload == "dense" and world > 1 and args.scaling == "strong" and not args.no_weak:
        # the north star's multi-GPU target is weak scaling: the same line also times a fixed
        # 65536-row slab per GPU (m = N x 65536; device-timed only). Its value is the whole job's
        # it/s, so weak-scaling efficiency = weak.value / value at N = 1.
        import copy

        wa = copy.copy(args)
        wa.scaling, wa.no_e2e, wa.no_cpu_baseline = "weak", True, True
        wk = run_workload(wa, "dense", args.m, args.n, k, K, W, env)
        if out is not None and wk is not None:
            out["weak"] = {key: wk[key] for key in ("value", "unit", "ms_per_step", "scaling", "config", "roofline",
                                                    "gpu_launches") if key in wk}
    # BASELINE.json's metric is "dense+sparse": the default dense line carries config 3 too
    if args.workload == "dense" and not args.no_sparse:
        if comm is None:
            ctx.close()
            ctx = nmf.Context(local)
            env["ctx"] = ctx
        sp = run_workload(args, "sparse", 1 << 22, 1 << 22, 32, K, W, env)
        if out is not None:
            out["sparse"] = sp
    if rank == 0:
        emit(out)
    if comm:
        comm.close()
        torch.distributed.destroy_process_group()
    else:
        ctx.close()


def run_workload(args, workload, m, n, k, K, W, env):
    nmf, np, torch, ctx = env["nmf"], env["np"], env["torch"], env["ctx"]
    rank, world, local = env["rank"], env["world"], env["local"]
    barrier, max_over_ranks, sum_over_ranks = env["barrier"], env["max_over_ranks"], env["sum_over_ranks"]
    kp = 8 if k <= 8 else 16 if k <= 16 else 32 if k <= 32 else 64
    hbm, peak_src = peaks()
    extra = {}
    host_buf = None

    # ------------------------------------------------------------------ set up A
    weak = args.scaling == "weak" and workload != "ooc"
    if workload == "ooc":
        rows_per_rank = m // world if m else int(args.ooc_gb * 1e9 / (n * 4)) // 128 * 128
        m = rows_per_rank * world
    elif weak:
        m = m * world  # weak scaling: a fixed slab per GPU (the paper's [N x 65536, ...] pattern)
    plan = nmf.make_plan(m, n, k, world, 1, nmf.Strategy.rnmf)
    (r0, r1), _ = plan.slabs[rank]
    rows = r1 - r0
    t_setup = time.perf_counter()
    density = args.density
    if workload == "dense":
        ctx.set_problem(m, n, k, r0, rows)
        ctx.generate_dense_uniform(42, 99)
        wl = f"dense synthetic {m}x{n} f32 uniform A (CounterRng(42,99)), k={k}, RNMF row slabs"
        metric = f"MU iters/sec (dense {m}x{n}, k={k}, 1D row-partitioned, NCCL all-reduce)"
        # one streaming pass reads the A slab once plus its factor operand and output
        # (SURVEY.md §8(d)); the one-pass kernel reads A from HBM once for both contractions
        bytes_per_launch = {"aht_pass (A.H^T)": rows * n * 4 + (n + rows) * k * 4,
                            "wta_pass (A^T.W)": rows * n * 4 + (n + rows) * k * 4,
                            # the iteration's algorithmic work is both A passes,
                            # 2 |A_slab|; the one-pass kernel does both (the second from L2)
                            FUSED: 2 * rows * n * 4 + 2 * (n + rows) * k * 4}
    elif workload == "sparse":
        ctx.set_problem(m, n, k, r0, rows)
        ctx.generate_csr_uniform(density, 1)
        import ctypes as C

        cnt = C.c_uint64()
        nmf.check(nmf._capi.lib().oocnmf_csr_nnz(ctx._h, C.byref(cnt)))
        nnz = int(cnt.value)
        wl = (f"sparse synthetic CSR {m}x{n}, density {density} (reference generator "
              f"synth.cpp:60-86 on device, seed 1), nnz/rank={nnz}, k={k}, RNMF row slabs")
        metric = f"MU iters/sec (sparse CSR {m}x{n} density {density}, k={k}, 1D row-partitioned)"
        # gather model: CSR (8 B/nnz) + row_ptr + one kp-wide factor row per
        # nonzero + output, per SpMM; pass 2 runs on CSR(A^T) (n rows)
        bytes_per_launch = {"aht_pass (A.H^T)": nnz * 8 + (rows + 1) * 8 + nnz * kp * 4 + rows * kp * 4,
                            "wta_pass (A^T.W)": nnz * 8 + (n + 1) * 8 + nnz * kp * 4 + n * kp * 4}
        extra["nnz_per_rank"] = nnz
    else:
        # out-of-core: A slab in pinned host memory, generated on the device in chunks
        ctx.set_problem(m, n, k, r0, rows)
        host_buf = np.empty((rows, n), np.float32)
        nmf.check(nmf._capi.lib().oocnmf_host_register(host_buf.ctypes.data, host_buf.nbytes))
        chunk = max(128, (8 << 30) // (n * 4) // 128 * 128)
        with nmf.Context(local) as gen:
            for c0 in range(0, rows, chunk):
                cr = min(chunk, rows - c0)
                gen.set_problem(m, n, k, r0 + c0, cr)
                gen.generate_dense_uniform(42, 99)
                gen.download_dense(host_buf[c0:c0 + cr])
        ctx.attach_host(host_buf)
        wl = (f"out-of-core dense {m}x{n} f32 uniform A, {rows * n * 4 / 1e9:.1f} GB pinned host slab/rank "
              f"(config 4 scaled to this host's RAM), k={k}, streamed every iteration")
        metric = f"MU iters/sec (out-of-core dense {m}x{n}, k={k}, host-link streaming)"
        bytes_per_launch = rows * n * 4
    extra["setup_s"] = time.perf_counter() - t_setup

    # ------------------------------------------------------------------ timed solve
    ctx.solve(nmf.NmfConfig(k=k, max_iters=W, error_check_interval=W, eta=0.0, seed=0))
    cfg = nmf.NmfConfig(k=k, max_iters=K, error_check_interval=10, eta=0.0, init=nmf.FactorInit.resident)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        trace, info = ctx.solve(cfg)
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    value = K / (ms / 1e3)

    traffic = None  # ncu dram bytes per launch of the dominant kernel, when captured for this config
    prof = os.path.join(ROOT, "profiles", "ncu_dram_per_launch.json")
    if world == 1 and os.path.exists(prof):
        if workload == "dense" and (m, n, k) == (65536, 65536, 32):
            traffic = json.load(open(prof))
        elif workload == "sparse" and (m, n, k) == (1 << 22, 1 << 22, 32) and density == 1e-5:
            traffic = json.load(open(prof)).get("sparse")
    if workload == "ooc":
        # host-link roofline: measured pinned H2D bandwidth on this GPU (concurrently on all ranks)
        probe = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        dev = torch.empty_like(probe, device="cuda")
        for _ in range(2):
            dev.copy_(probe, non_blocking=True)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(8):
            dev.copy_(probe, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        link = 8 * probe.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9
        link = min(link, max_over_ranks(link)) if world == 1 else -max_over_ranks(-link)
        achieved = rows * n * 4 * value / 1e9
        roof = {"bound": "host-link", "achieved": achieved, "peak": link, "unit": "GB/s", "frac": achieved / link,
                "traffic": None, "kernel": "row-batch sweep (H2D copy stream, overlapped compute)",
                "algorithmic_bytes_per_launch": rows * n * 4, "avg_launch_ms": ms / K,
                "peak_source": "measured pinned H2D (torch copy_ of a 1 GiB pinned buffer, 8 reps) on this box",
                "hbm_pass_ms": {"aht_pass (A.H^T)": info["aht_pass_ms"] / max(1, info["aht_pass_launches"]),
                                "wta_pass (A^T.W)": info["wta_pass_ms"] / max(1, info["wta_pass_launches"])}}
    else:
        roof = roofline(info, bytes_per_launch, hbm, peak_src, traffic)
        if workload == "sparse":
            roof["note"] = ("both passes are k_spmm_mu launches: the SpMM with the factor update fused into it "
                            "(A.H^T + W update; A^T.W + H update except on error-check iterations, single rank); "
                            "the algorithmic bytes count the SpMM only")
    extra["a_pass_gbs_total"] = sum_over_ranks(2 * rows * n * 4 * value / 1e9) if workload == "dense" else None

    # ------------------------------------------------------------------ e2e through the public API
    e2e = None
    if not args.no_e2e and workload in ("dense", "sparse"):
        e2e = e2e_runs(args, workload, m, n, k, K, rows, r0, kp, env)
    elif workload == "ooc":
        e2e = {"value": value, "unit": "it/s", "h2d_bytes_per_step": rows * n * 4, "d2h_bytes_per_step": 16,
               "note": "out-of-core: the timed solve already reads A from pinned host memory every iteration"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if workload == "dense":
            _, cpu = cpu_reference_dense(m, n, k, args.cpu_seconds)
        elif workload == "sparse":
            samples = []
            for sr in (2048, 65536):  # a wide row range keeps the per-row slope above the noise
                with nmf.Context(local) as g:
                    g.set_problem(m, n, k, 0, sr)
                    g.generate_csr_uniform(density, 1)
                    samples.append((sr, g.download_csr()))
            _, cpu = cpu_reference_sparse(samples, m, k, args.cpu_seconds)

    if host_buf is not None:
        ctx.set_problem(m, n, k, r0, rows)  # detach the host slab before unregistering it
        nmf._capi.lib().oocnmf_host_unregister(host_buf.ctypes.data)
    if rank != 0:
        return None
    out = {"metric": metric, "value": value, "unit": "it/s", "n_gpus": world, "steps": K, "warmup": W,
           "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak" if weak else "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": wl, "m": m, "n": n, "k": k, "parallelism": f"rnmf-dp{world}",
                      "rows_per_rank": rows, "error_check_interval": 10,
                      "l2": f"A slab >> 126 MB L2 (no flush needed)"},
           "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
           "gpu_launches": int(info["gpu_launches"]), "paths": ctx.paths(),
           "final_rel_error": trace[-1][1] if trace else None,
           "phase_ms_per_step": {p_: info[p_ + "_s"] * 1e3 / K for p_ in
                                 ("w_update", "h_update", "allreduce", "error_check")}}
    out.update({k_: v for k_, v in extra.items() if v is not None})
    return out


def e2e_runs(args, workload, m, n, k, K, rows, r0, kp, env):
    """End to end through the public API on HOST buffers, K iterations, every phase timed with
    the device synchronised at its end (phases sum to the total): context creation, A upload
    (host -> device, narrowing / layout on the device), the solve, the factor download
    (device -> host, f64 reference layouts), context destruction.

    Two runs: the headline uses the library's f32 extension on page-locked host memory
    (oocnmf_load_dense_f32 / the CSR upload); the second is the reference-shaped call, an f64
    pageable row-major A handed to nmf_serial exactly as a reference caller holds it
    (include/oocnmf/nmf.hpp:64 via MatrixRef(DenseMatrix)), dense at N = 1 only (34 GB)."""
    nmf, np, torch = env["nmf"], env["np"], env["torch"]
    world, local, barrier, max_over_ranks = env["world"], env["local"], env["barrier"], env["max_over_ranks"]
    ctx = env["ctx"]
    if workload == "dense":
        host = np.empty((rows, n), np.float32)
        ctx.download_dense(host)
        h2d = rows * n * 4
    else:
        host = ctx.download_csr()
        h2d = host.nnz * 12 + (rows + 1) * 8
    d2h = rows * k * 8 + k * n * 8 + 16 * (K // 10 + 1)
    ecfg = nmf.NmfConfig(k=k, max_iters=K, error_check_interval=10, eta=0.0, seed=0, device=local)

    def one(a_host, use_comm_ctx):
        ph = {}
        # Python's cyclic GC freeing earlier multi-GB arrays (munmap) must not land inside a
        # phase: collect now, pause it for the timed call (re-enabled in e2e_runs)
        gc.collect()
        gc.disable()
        barrier()
        t0 = time.perf_counter()
        t = t0
        c = ctx if use_comm_ctx else nmf.Context(local)

        def mark(name):
            nonlocal t
            torch.cuda.synchronize()
            now = time.perf_counter()
            ph[name] = now - t
            t = now
        mark("create")
        c.set_problem(m, n, k, r0, rows)
        if workload == "dense":
            c.load_dense(a_host)
        else:
            c.load_csr(a_host)
        mark("upload")
        c.solve(ecfg)
        mark("solve")
        c.get_factors()
        if world > 1:
            c.gather_w()
        mark("download")
        if not use_comm_ctx:
            c.close()
        mark("destroy")
        total = max_over_ranks(time.perf_counter() - t0)
        return total, {k_: round(v, 4) for k_, v in ph.items()}

    pinned = workload == "dense"
    if pinned:
        nmf.check(nmf._capi.lib().oocnmf_host_register(host.ctypes.data, host.nbytes))
    try:
        total, ph = one(host, world > 1)
    finally:
        gc.enable()
        if pinned:
            nmf._capi.lib().oocnmf_host_unregister(host.ctypes.data)
    e2e = {"value": K / total, "unit": "it/s", "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
           "phases_s": ph, "total_s": total,
           "note": f"public API on host buffers: A ({h2d / 1e9:.2f} GB/rank, "
                   f"{'f32 page-locked' if pinned else 'CSR u64/f64 pageable'}) uploaded once, {K} iterations, "
                   f"W/H downloaded as f64; phases sum to total_s"}
    if workload == "dense" and world == 1 and not args.no_e2e_f64:
        a64 = host.astype(np.float64)
        del host
        try:
            t64, ph64 = one(a64, False)
        finally:
            gc.enable()
        e2e["reference_shaped"] = {"value": K / t64, "unit": "it/s", "h2d_bytes_per_step": a64.nbytes / K,
                                   "d2h_bytes_per_step": d2h / K, "phases_s": ph64, "total_s": t64,
                                   "note": "f64 pageable row-major A as a reference caller holds it "
                                           "(nmf_serial(MatrixRef(DenseMatrix))): staged copy-in, narrowing to f32 "
                                           "on the device"}
    return e2e


if __name__ == "__main__":
    _quiet_stdout()
    main()
