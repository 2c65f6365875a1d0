"""The oocnmf command-line front end on the GPU (paper_2202_09518_b200/cli/oocnmf_cli.cpp, the
reference's tools/oocnmf_cli.cpp): `factorize` writes the reference's run
outputs (w.pdn1, h.pdn1, error_trace.csv, counters.json, stats.json, manifest.json,
oocnmf_cli.cpp:166-195) with factors and trace matching the compiled reference, in core, out of
core from a PDN1 file under --budget, over threads and over the tcp backend (--spawn-local);
`select-k` writes selection.json / .csv matching the reference's select_k; `bench` emits the
long-form phase CSV (:336-373); `gen --type sparse` is byte-identical to the reference's
generator."""
import csv
import io
import json
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_2202_09518_b200 as nmf

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not oracle.ref.available, reason="needs oracle/_ref")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2202_09518_b200", "bin", "oocnmf")
TRACE_TOL, FACTOR_TOL = 1e-4, 1e-3


def run(*args, cwd=None, timeout=600):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=timeout)
    return r


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _input(tmp_path, m=600, n=400, kt=6, name="a.pdn1"):
    """A low-rank A (reference generator), f32-rounded so the GPU (f32 storage) and the reference
    (f64) see the same matrix, written with the reference's own PDN1 writer."""
    a = oracle.ref.gen_lowrank(m, n, kt, 0.05, 21)[0].astype(np.float32).astype(np.float64)
    oracle.ref.write_pdn1(tmp_path / name, a)
    return a


def _read_trace(path):
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["iteration", "relative_error"]
    return [int(r[0]) for r in rows[1:]], np.array([float(r[1]) for r in rows[1:]])


def _check_outputs(out, ref, k, expect_iters):
    it, err = _read_trace(out / "error_trace.csv")
    assert it == [i for i, _ in ref.error_trace] and it[-1] == expect_iters
    np.testing.assert_allclose(err, [e for _, e in ref.error_trace], rtol=TRACE_TOL)
    w, h = oracle.ref.read_matrix(out / "w.pdn1"), oracle.ref.read_matrix(out / "h.pdn1")
    assert w.shape == ref.w.shape and h.shape == ref.h.shape
    assert rel_fro(w, ref.w) <= FACTOR_TOL and rel_fro(h, ref.h) <= FACTOR_TOL
    return it, err


@needs_ref
def test_factorize_writes_the_reference_outputs(gpu, tmp_path):
    a = _input(tmp_path)
    r = run("factorize", "--input", tmp_path / "a.pdn1", "--k", 6, "--eta", 0, "--max-iters", 60, "--seed", 3,
            "--out", tmp_path / "out")
    assert r.returncode == 0, r.stderr
    out = tmp_path / "out"
    ref = oracle.ref.nmf_serial(a, 6, max_iters=60, interval=10, eta=0.0, seed=3)
    it, err = _check_outputs(out, ref, 6, 60)
    summary = json.loads(r.stdout.strip().splitlines()[-1])
    assert summary == {"converged": False, "final_error": float(err[-1]), "iterations": 60, "out": str(out)}

    counters = json.loads((out / "counters.json").read_text())
    assert sorted(counters) == sorted(["w_update_s", "h_update_s", "allreduce_s", "error_check_s", "io_s",
                                       "total_s", "flops", "peak_resident_bytes"])
    assert counters["total_s"] > 0 and counters["flops"] > 0
    stats = json.loads((out / "stats.json").read_text())
    assert set(stats["per_tag"]) == {"generic", "w_update", "h_update", "error_check", "gather", "barrier"}
    assert set(stats) == {"per_tag", "total_bytes", "total_calls", "total_seconds"}

    text = (out / "manifest.json").read_text()
    man = json.loads(text)
    assert man["command"] == "factorize" and man["version"] == "oocnmf 1.0.0"
    assert man["config"] == {"input": str(tmp_path / "a.pdn1"), "k": 6, "eta": 0.0, "max_iters": 60, "workers": 1,
                             "backend": "threads", "batches": 1, "budget": 0, "strategy": "auto", "seed": 3}
    assert man["plan"] == json.loads(oracle.ref.plan_to_json(600, 400, 6, 1, 1, 0))
    assert man["outputs"] == {k: str(out / v) for k, v in (("w", "w.pdn1"), ("h", "h.pdn1"),
                                                            ("error_trace", "error_trace.csv"),
                                                            ("counters", "counters.json"))}
    assert man["result"] == {"iterations_run": 60, "converged": False, "final_error": float(err[-1])}
    # every JSON file is laid out byte for byte as the reference's nlohmann dump(2) would write it
    for name in ("manifest.json", "counters.json", "stats.json"):
        t = (out / name).read_text()
        assert t.endswith("}\n") and oracle.ref.json_reformat(t, 2) + "\n" == t, name


@needs_ref
def test_factorize_stops_at_eta_like_the_reference(gpu, tmp_path):
    a = _input(tmp_path, 300, 200, 4)
    r = run("factorize", "--input", tmp_path / "a.pdn1", "--k", 4, "--eta", 0.05, "--max-iters", 400,
            "--out", tmp_path / "o")
    assert r.returncode == 0, r.stderr
    ref = oracle.ref.nmf_serial(a, 4, max_iters=400, interval=10, eta=0.05, seed=0)
    assert ref.converged and ref.iterations_run < 400
    _check_outputs(tmp_path / "o", ref, 4, ref.iterations_run)
    man = json.loads((tmp_path / "o" / "manifest.json").read_text())
    assert man["result"]["converged"] and man["result"]["iterations_run"] == ref.iterations_run


@needs_ref
def test_factorize_out_of_core_from_file_under_budget(gpu, tmp_path):
    _input(tmp_path, 1000, 300, 5)
    base = run("factorize", "--input", tmp_path / "a.pdn1", "--k", 5, "--eta", 0, "--max-iters", 30,
               "--out", tmp_path / "incore")
    # a 300 KB budget: the 2.4 MB file streams in row batches (ASource::file + StoreConfig,
    # oocnmf_cli.cpp:239-242)
    ooc = run("factorize", "--input", tmp_path / "a.pdn1", "--k", 5, "--eta", 0, "--max-iters", 30,
              "--budget", 300000, "--out", tmp_path / "ooc")
    assert base.returncode == 0 and ooc.returncode == 0, ooc.stderr
    _, e1 = _read_trace(tmp_path / "incore" / "error_trace.csv")
    _, e2 = _read_trace(tmp_path / "ooc" / "error_trace.csv")
    np.testing.assert_allclose(e2, e1, rtol=1e-6)
    w1, w2 = oracle.ref.read_matrix(tmp_path / "incore" / "w.pdn1"), oracle.ref.read_matrix(tmp_path / "ooc" / "w.pdn1")
    assert rel_fro(w2, w1) < 1e-5
    man = json.loads((tmp_path / "ooc" / "manifest.json").read_text())
    assert man["config"]["budget"] == 300000


def _workers():
    return max(1, min(nmf.device_count(), 4))


@needs_ref
@pytest.mark.parametrize("backend", ["threads", "tcp"])
def test_factorize_distributed_backends(gpu, tmp_path, backend):
    """--workers N over the threads backend (run_distributed_threads) and over the tcp backend
    with --spawn-local (one process per rank, NCCL bootstrapped by connect_tcp); one GPU per
    rank (a one-GPU box runs N = 1 through the same code)."""
    n_w = _workers()
    a = _input(tmp_path, 800, 500, 5)
    extra = ["--spawn-local", 1] if backend == "tcp" else []
    r = run("factorize", "--input", tmp_path / "a.pdn1", "--k", 5, "--eta", 0, "--max-iters", 40,
            "--workers", n_w, "--backend", backend, "--strategy", "rnmf", "--out", tmp_path / "o", *extra)
    assert r.returncode == 0, r.stderr
    ref = oracle.ref.nmf_distributed(a, 5, n_w, strategy=2, max_iters=40, interval=10, eta=0.0, seed=0)
    _check_outputs(tmp_path / "o", ref, 5, 40)
    man = json.loads((tmp_path / "o" / "manifest.json").read_text())
    assert man["config"]["workers"] == n_w and man["config"]["backend"] == backend
    assert len(man["plan"]["workers"]) == n_w
    stats = json.loads((tmp_path / "o" / "stats.json").read_text())
    if n_w > 1:
        assert stats["per_tag"]["h_update"]["calls"] == 40 and stats["total_bytes"] > 0


@needs_ref
def test_select_k_writes_the_reference_selection(gpu, tmp_path):
    a = oracle.ref.gen_lowrank(120, 90, 3, 0.01, 14)[0].astype(np.float32).astype(np.float64)
    oracle.ref.write_pdn1(tmp_path / "a.pdn1", a)
    r = run("select-k", "--input", tmp_path / "a.pdn1", "--k-min", 1, "--k-max", 4, "--perturbations", 6,
            "--eta", 0, "--max-iters", 300, "--seed", 5, "--out", tmp_path / "sel")
    assert r.returncode == 0, r.stderr
    recs, chosen, _, why = oracle.ref.select_k(a, 1, 4, n_perturbations=6, delta=0.03, sil_threshold=0.75,
                                               max_iters=300, interval=10, eta=0.0, seed=5)
    js = (tmp_path / "sel" / "selection.json").read_text()
    assert r.stdout == js
    got = json.loads(js)
    assert got["chosen_k"] == (chosen if chosen is not None else "none")
    for g, w in zip(got["records"], recs):
        assert (g["k"], g["valid"], g["runs_used"]) == (w["k"], w["valid"], w["runs_used"])
        assert g["mean_relative_error"] == pytest.approx(w["mean_relative_error"], rel=1e-4)
        assert g["min_silhouette"] == pytest.approx(w["min_silhouette"], abs=1e-4)
    # file bytes: the reference's to_json / to_csv of the same records
    ref_js, ref_csv = oracle.ref.selection_json_csv(got["records"], None if got["chosen_k"] == "none"
                                                    else got["chosen_k"], got["rationale"])
    assert js == ref_js + "\n"
    assert (tmp_path / "sel" / "selection.csv").read_text() == ref_csv
    bad = run("select-k", "--input", tmp_path / "a.pdn1", "--k-min", 5, "--k-max", 2)
    assert bad.returncode == 2 and json.loads(bad.stderr)["error"]["type"] == "usage"


def test_bench_emits_the_long_form_phase_csv(gpu, tmp_path):
    workers = [1] + ([2] if nmf.device_count() >= 2 else [])
    r = run("bench", "--rows", 512, "--cols", 384, "--k", 4, 8, "--workers", *workers, "--iters", 5,
            "--out", tmp_path / "b.csv")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO((tmp_path / "b.csv").read_text())))
    assert len(rows) == 12 * len(workers)
    assert [x["phase"] for x in rows[:6]] == ["w_update", "h_update", "allreduce", "error_check", "io", "total"]
    for x in rows:
        assert x["strategy"] == "rnmf" and x["N"] in map(str, workers) and x["n_B"] == "1" and x["k"] in ("4", "8")
        assert float(x["seconds"]) >= 0 and int(x["bytes"]) >= 0
    if len(workers) > 1:  # the two-rank rows carry the all-reduced bytes (CollectiveStats)
        assert all(int(x["bytes"]) > 0 for x in rows if x["N"] == "2" and x["phase"] == "total")
    assert all(float(x["seconds"]) > 0 for x in rows if x["phase"] == "total")
    r = run("bench", "--rows", 256, "--cols", 256, "--k", 4, "--workers", 1, "--iters", 2)
    assert r.returncode == 0 and r.stdout.startswith("strategy,N,n_B,k,phase,seconds,bytes\n")


@needs_ref
@pytest.mark.parametrize("ext", ["pdn1", "mtx"])
def test_gen_sparse_is_byte_identical_to_the_reference(gpu, tmp_path, ext):
    m, n, dens, seed = 300, 500, 0.02, 4
    r = run("gen", "--type", "sparse", "--rows", m, "--cols", n, "--density", dens, "--seed", seed,
            "--out", f"s.{ext}", cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    rp, ci, v, shape = oracle.ref.gen_sparse(m, n, dens, seed)
    writer = oracle.ref.write_pdn1 if ext == "pdn1" else oracle.ref.write_mtx
    writer(tmp_path / f"r.{ext}", (rp, ci, v, shape))
    assert (tmp_path / f"s.{ext}").read_bytes() == (tmp_path / f"r.{ext}").read_bytes()


@needs_ref
def test_factorize_tcp_with_explicit_peers(gpu, tmp_path):
    """--backend tcp --rank r --peers host:port: one process per rank started by the caller (the
    multi-host form, oocnmf_cli.cpp:273-274), here two processes on two GPUs of this box."""
    if nmf.device_count() < 2:
        pytest.skip("needs two GPUs")
    a = _input(tmp_path, 640, 384, 4)
    port = 20000 + os.getpid() % 20000
    args = ["factorize", "--input", tmp_path / "a.pdn1", "--k", 4, "--eta", 0, "--max-iters", 30, "--workers", 2,
            "--backend", "tcp", "--strategy", "rnmf", "--peers", f"127.0.0.1:{port}", "--out", tmp_path / "o"]
    procs = []
    for r in (0, 1):
        env = dict(os.environ, OOCNMF_DEVICE=str(r))
        procs.append(subprocess.Popen([CLI, *map(str, args), "--rank", str(r)], stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True, env=env))
    outs = [p.communicate(timeout=300) for p in procs]
    assert [p.returncode for p in procs] == [0, 0], outs
    assert json.loads(outs[0][0].strip().splitlines()[-1])["iterations"] == 30
    assert outs[1][0].strip() == "" or "final_error" not in outs[1][0]  # only rank 0 reports
    ref = oracle.ref.nmf_distributed(a, 4, 2, strategy=2, max_iters=30, interval=10, eta=0.0, seed=0)
    _check_outputs(tmp_path / "o", ref, 4, 30)
