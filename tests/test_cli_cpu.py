"""CPU tests of the oocnmf command-line front end (paper_2202_09518_b200/cli/oocnmf_cli.cpp, the
reference's tools/oocnmf_cli.cpp) and of the host core's JSON output: argument handling and exit
codes, `gen --type lowrank` byte-identical to the reference's generator + writers, `--dump-plan`
identical to the reference's PartitionPlan::to_json, and the JSON writer (csrc/json_out.hpp,
SelectionReport::to_json / to_csv) byte-identical to the nlohmann library the reference is
compiled against. Nothing here touches a GPU."""
import json
import os
import struct
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2202_09518_b200", "bin", "oocnmf")
LIB = os.path.join(ROOT, "paper_2202_09518_b200", "lib")
needs_ref = pytest.mark.skipif(not oracle.ref.available, reason="needs oracle/_ref")


def run(*args, cwd=None, env=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=120, env=env)


@pytest.fixture(scope="module")
def json_demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("jd") / "json_demo")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(ROOT, "paper_2202_09518_b200", "csrc"), os.path.join(ROOT, "tests", "cpp", "json_demo.cpp"),
                    "-L", LIB, "-loocnmf_b200", "-Wl,-rpath," + LIB, "-o", exe], check=True)
    return exe


def test_version_help_and_usage_errors():
    r = run("--version")
    assert r.returncode == 0 and r.stdout.strip() == "oocnmf 1.0.0"
    r = run("--help")
    assert r.returncode == 0 and "factorize" in r.stdout and "select-k" in r.stdout
    r = run("factorize", "--help")
    assert r.returncode == 0 and "--spawn-local" in r.stdout and "--dump-plan" in r.stdout
    # parse errors: message + exit 2 (CLI11's behaviour in oocnmf_cli.cpp:439-445)
    for args in ([], ["frobnicate"], ["factorize", "--k", "3"], ["gen", "--rows", "4", "--cols", "x", "--out", "a"],
                 ["factorize", "--input", "a", "--k", "3", "--backend", "mpi"], ["bench", "--rows", "4", "--cols", "4",
                                                                                 "--k", "2", "--workers"]):
        r = run(*args)
        assert r.returncode == 2, (args, r.stderr)
        assert "Run with --help" in r.stderr
    # usage failures inside a command: {"error": {...}} on stderr, exit 2 (oocnmf_cli.cpp:52-58)
    r = run("factorize", "--input", "/nonexistent.pdn1", "--k", "3")
    assert r.returncode == 2
    assert json.loads(r.stderr) == {"error": {"message": "input file not found: /nonexistent.pdn1", "type": "usage"}}
    assert r.stderr.startswith('{"error":{"message":')  # compact dump, sorted keys


@needs_ref
@pytest.mark.parametrize("noise", [0.0, 0.2])
def test_gen_lowrank_is_byte_identical_to_the_reference(tmp_path, noise):
    m, n, kt, seed = 97, 61, 5, 13
    r = run("gen", "--rows", m, "--cols", n, "--k-true", kt, "--noise", noise, "--seed", seed, "--out", "a.pdn1",
            "--out-w0", "w0.mtx", "--out-h0", "h0.pdn1", cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout) == {"written": "a.pdn1"}
    a, w0, h0 = oracle.ref.gen_lowrank(m, n, kt, noise, seed)
    oracle.ref.write_pdn1(tmp_path / "ra.pdn1", a)
    oracle.ref.write_mtx(tmp_path / "rw0.mtx", w0)
    oracle.ref.write_pdn1(tmp_path / "rh0.pdn1", h0)
    for ours, theirs in (("a.pdn1", "ra.pdn1"), ("w0.mtx", "rw0.mtx"), ("h0.pdn1", "rh0.pdn1")):
        assert (tmp_path / ours).read_bytes() == (tmp_path / theirs).read_bytes(), ours
    r = run("gen", "--rows", 4, "--cols", 4, "--k-true", 5, "--out", "x.pdn1", cwd=tmp_path)
    assert r.returncode == 2 and "k_true must not exceed" in r.stderr


@needs_ref
@pytest.mark.parametrize("workers,batches,strategy", [(1, 1, "auto"), (3, 2, "rnmf"), (2, 3, "cnmf"), (4, 1, "auto")])
def test_dump_plan_is_the_reference_plan(tmp_path, workers, batches, strategy):
    m, n = 40, 70  # n > m: auto picks cnmf (partition.cpp:12-14)
    a = np.arange(m * n, dtype=np.float64).reshape(m, n) + 1
    oracle.ref.write_pdn1(tmp_path / "a.pdn1", a)
    r = run("factorize", "--input", tmp_path / "a.pdn1", "--k", 4, "--workers", workers, "--batches", batches,
            "--strategy", strategy, "--dump-plan")
    assert r.returncode == 0, r.stderr
    st = 1 if strategy == "cnmf" or (strategy == "auto" and n > m) else 0
    assert r.stdout == oracle.ref.plan_to_json(m, n, 4, workers, batches, st) + "\n"


def _hex(x):
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


@needs_ref
def test_json_numbers_match_nlohmann(json_demo):
    rng = np.random.default_rng(5)
    xs = [0.1, 0.5, 1.0, 2.0, 100.0, 1e15, 1e16, 1.5e16, 123456789012345.0, 1e-4, 1.2e-4, 1e-5, 9.99e-5,
          5e-324, 1.7976931348623157e308, 0.502504328195, 1 / 3, -2.5, -1e-7, 6.02e23, 2 ** 53, 0.001]
    xs += list(rng.random(200)) + list(10.0 ** rng.uniform(-30, 30, 300)) + list(-rng.random(50) * 1e-3)
    xs += list(np.round(rng.random(50) * 1000, 3))
    raw = rng.integers(0, 2 ** 63, 20000, dtype=np.uint64).view(np.float64)  # every exponent, subnormals
    xs += [float(x) for x in raw if np.isfinite(x)]
    xs += [float(x) for x in rng.random(5000).astype(np.float32)]  # f32-rounded values, as the solver reports
    out = subprocess.run([json_demo, "numbers"], input="\n".join(_hex(x) for x in xs), capture_output=True,
                         text=True, check=True).stdout.split("\n")
    out = out[:len(xs)]
    for x, s in zip(xs, out):
        assert float(s) == x, (x, s)  # round-trips
    doc = "[" + ",".join(out) + "]"
    ref = oracle.ref.json_reformat(doc, -1)
    if ref != doc:
        bad = [(x, s, r) for x, s, r in zip(xs, out, ref[1:-1].split(",")) if s != r]
        pytest.fail(f"{len(bad)} numbers differ from nlohmann, e.g. {bad[:5]}")


@needs_ref
def test_json_document_layout_matches_nlohmann(json_demo):
    out = subprocess.run([json_demo, "document"], capture_output=True, text=True, check=True).stdout
    pretty, compact = out[:-1].split("\n---\n")
    assert oracle.ref.json_reformat(pretty, 2) == pretty
    assert oracle.ref.json_reformat(pretty, -1) == compact


@needs_ref
@pytest.mark.parametrize("chosen", [None, 3])
def test_selection_report_json_and_csv_are_the_reference_bytes(json_demo, chosen):
    rng = np.random.default_rng(1)
    recs = [dict(k=k, valid=bool(k % 2), runs_used=16 - k, min_silhouette=float(rng.uniform(-1, 1)),
                 mean_silhouette=float(rng.random()), mean_relative_error=float(rng.random() * 1e-3))
            for k in range(2, 7)]
    recs[1]["min_silhouette"] = 0.75
    why = 'largest k with min silhouette >= 0.75 "quoted"'
    lines = [f"{len(recs)} {-1 if chosen is None else chosen}"]
    lines += [f"{r['k']} {int(r['valid'])} {r['runs_used']} {_hex(r['min_silhouette'])} {_hex(r['mean_silhouette'])} "
              f"{_hex(r['mean_relative_error'])}" for r in recs]
    out = subprocess.run([json_demo, "selection"], input="\n".join(lines + [why]) + "\n", capture_output=True,
                         text=True, check=True).stdout
    js, csv = out.split("\n---\n")
    ref_js, ref_csv = oracle.ref.selection_json_csv(recs, chosen, why)
    assert js == ref_js
    assert csv == ref_csv


@needs_ref
def test_tcp_backend_argument_errors(tmp_path):
    """--backend tcp without peers, and a malformed endpoint (connect_tcp, comm.hpp:84-87): usage
    errors (exit 2) raised before any device or socket work."""
    oracle.ref.write_pdn1(tmp_path / "a.pdn1", np.arange(1, 61, dtype=np.float64).reshape(6, 10))
    base = ["factorize", "--input", tmp_path / "a.pdn1", "--k", 2, "--workers", 2, "--backend", "tcp"]
    r = run(*base)
    assert r.returncode == 2
    assert json.loads(r.stderr)["error"] == {"message": "--backend tcp needs --peers or --spawn-local", "type": "usage"}
    r = run(*base, "--rank", 1, "--peers", "no-port-here")
    assert r.returncode == 2
    assert json.loads(r.stderr)["error"]["message"] == "endpoint must be host:port, got no-port-here"
    r = run(*base, "--rank", 5, "--peers", "127.0.0.1:1")
    assert r.returncode == 2 and json.loads(r.stderr)["error"]["message"] == "tcp rank out of range"
