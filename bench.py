#!/usr/bin/env python
"""Benchmark of the MU-NMF hot path (BASELINE.json metric: MU iters/sec and A-pass GB/s vs
the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload dense]

A "step" is one MU iteration (W update then H update, error every 10 iterations as the
reference default) over the synthetic dense 65536 x 65536 f32 A with k = 32 (config 2),
row-partitioned over N GPUs (strong scaling). One JSON line on rank 0.

--impl reference times the reference's own CPU solver (oracle/_ref, compiled from
/root/reference sources; the oracle port if absent) on this box's host cores, one MU
iteration per step on a bounded row sample, extrapolated to the full matrix (cost is
linear in rows).
"""
import argparse
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["dense"], default="dense")
    p.add_argument("--m", type=int, default=65536)
    p.add_argument("--n", type=int, default=65536)
    p.add_argument("--k", type=int, default=32)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = str(index)
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9 or f[0] != self.index:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_reference_rate(m, n, k, seconds, steps=None, warmup=0):
    """Reference CPU solver, one MU iteration per step on a row sample; returns (it/s
    extrapolated to m rows, dict)."""
    import numpy as np

    import oracle

    impl = oracle.ref if oracle.ref.available else oracle.port
    kind = "reference" if impl is oracle.ref else "port"
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


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    m, n, k, K, W = args.m, args.n, args.k, args.steps, max(3, args.warmup)
    workload = f"dense synthetic {m}x{n} f32 uniform A (CounterRng(42,99)), k={k}, RNMF row slabs"
    metric = f"MU iters/sec (dense {m}x{n}, k={k}, 1D row-partitioned, NCCL all-reduce)"

    if args.impl == "reference":
        if rank != 0:
            return
        rate, cb = cpu_reference_rate(m, n, k, args.cpu_seconds, steps=K, warmup=W)
        cb["sample"] = cb["sample"].replace("MU iterations", f"timed MU iterations after {W} warm-up")
        print(json.dumps({"impl": "reference", "metric": metric, "value": rate, "unit": "it/s", "n_gpus": args.gpus,
                          "steps": K, "warmup": W, "ms_per_step": 1e3 / rate, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": workload, "m": m, "n": n, "k": k, "parallelism": "host cores"},
                          "cpu_baseline": cb,
                          "e2e": {"value": rate, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import numpy as np
    import torch

    import paper_2202_09518_b200 as nmf

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    plan = nmf.make_plan(m, n, k, world, 1, nmf.Strategy.rnmf)
    (r0, r1), _ = plan.slabs[rank]
    rows = r1 - r0
    comm = nmf.DistComm(rank, world, local) if world > 1 else None
    ctx = comm.ctx if comm else nmf.Context(local)
    ctx.set_problem(m, n, k, r0, rows)
    ctx.generate_dense_uniform(42, 99)

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

    # warm-up: W iterations from the seeded init
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
    hbm, peak_src = peaks()

    # dominant streaming kernel: algorithmic bytes per launch / its CUDA-event duration
    per = {}
    for name, key in (("aht_pass (A.H^T)", "aht_pass_ms"), ("wta_pass (A^T.W)", "wta_pass_ms")):
        launches = max(1, int(info[key.replace("_ms", "_launches")]))
        per[name] = info[key] / launches
    dom = max(per, key=per.get)
    bytes_per_launch = rows * n * 4 + (n + rows) * k * 4
    achieved = bytes_per_launch / (per[dom] * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_dram_per_launch.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(dom.split()[0])
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": dom, "algorithmic_bytes_per_launch": bytes_per_launch,
                "avg_launch_ms": per[dom], "per_kernel_ms": per, "peak_source": peak_src}
    a_pass_gbs = 2 * m * n * 4 * value / 1e9  # whole-job A traffic, both passes

    # ---- e2e: host buffers through the public API, H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        host = np.empty((rows, n), np.float32)
        ctx.download_dense(host)
        nmf.check(nmf._capi.lib().oocnmf_host_register(host.ctypes.data, host.nbytes))
        try:
            barrier()
            t0 = time.perf_counter()
            if world == 1:
                import ctypes as C

                c = nmf.NmfConfig(k=k, max_iters=K, error_check_interval=10, eta=0.0, seed=0).to_c()
                wout, hout = np.empty((rows, k)), np.empty((k, n))
                ti, te = np.zeros(K // 10 + 2, np.uint64), np.zeros(K // 10 + 2)
                inf = nmf._capi.Info()
                nmf.check(nmf._capi.lib().oocnmf_nmf_serial_dense_f32(
                    local, host.ctypes.data_as(C.POINTER(C.c_float)), rows, n, C.byref(c),
                    None, None, wout.ctypes.data_as(C.POINTER(C.c_double)), hout.ctypes.data_as(C.POINTER(C.c_double)),
                    ti.ctypes.data_as(C.POINTER(C.c_uint64)), te.ctypes.data_as(C.POINTER(C.c_double)), ti.size,
                    C.byref(inf)))
            else:
                ctx.set_problem(m, n, k, r0, rows)
                ctx.load_dense(host)
                ctx.solve(nmf.NmfConfig(k=k, max_iters=K, error_check_interval=10, eta=0.0, seed=0))
                ctx.get_factors()
                ctx.gather_w()
            torch.cuda.synchronize()
            e2e_s = max_over_ranks(time.perf_counter() - t0)
        finally:
            nmf._capi.lib().oocnmf_host_unregister(host.ctypes.data)
        kp = 8 if k <= 8 else 16 if k <= 16 else 32 if k <= 32 else 64
        d2h = (((rows + 127) // 128 * 128) + (n + 127) // 128 * 128) * kp * 4 + 16 * (K // 10 + 1)
        e2e = {"value": K / e2e_s, "unit": "it/s", "h2d_bytes_per_step": rows * n * 4 / K,
               "d2h_bytes_per_step": d2h / K,
               "note": f"one public-API solve of {K} iterations on host (pinned) f32 buffers: A uploaded once "
                       f"({rows * n * 4 / 1e9:.2f} GB/rank), W/H downloaded once; bytes are per step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        _, cpu = cpu_reference_rate(m, n, k, args.cpu_seconds)

    if rank == 0:
        out = {"metric": metric, "value": value, "unit": "it/s", "n_gpus": world, "steps": K, "warmup": W,
               "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f32", "data": "synthetic",
               "config": {"workload": workload, "m": m, "n": n, "k": k, "parallelism": f"rnmf-dp{world}",
                          "rows_per_rank": rows, "error_check_interval": 10,
                          "l2": f"A slab {rows * n * 4 / 1e9:.1f} GB/rank >> 126 MB L2 (no flush needed)"},
               "a_pass_gbs": a_pass_gbs, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "clocks": clk.summary(), "gpu_launches": int(info["gpu_launches"]),
               "final_rel_error": trace[-1][1] if trace else None}
        print(json.dumps(out))
    if comm:
        comm.close()
        torch.distributed.destroy_process_group()
    else:
        ctx.close()


if __name__ == "__main__":
    main()
