"""bench.py contract on the CPU: the reference arm (the compiled reference, oracle/_ref, on the
host cores) prints exactly one JSON line on stdout with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_built():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libref_oocnmf.so"))


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mode", ["full", "sample"])
def test_reference_arm_prints_one_json_line(mode):
    # full: the same-config path (the whole A, nmf_serial with its checks) on a small A;
    # sample: the row-sample extrapolation used when the host cannot hold the f64 A
    extra = ["--m", "2048", "--n", "1024"] if mode == "full" else ["--ref-sample", "--cpu-seconds", "1"]
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "12",
                        "--warmup", "3"] + extra, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["unit"] == "it/s" and d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["same_config"] == (mode == "full")
    if mode == "full":
        assert d["config"]["m"] == 2048 and 0 < d["final_rel_error"] < 1


def test_clock_sampler_counts_only_timed_region_samples():
    """bench.ClockSampler.summary keeps the NVML samples taken after the timed region opened and
    decodes the throttle bits the contract names (hw_slowdown 0x8, hw_thermal 0x40,
    sw_thermal 0x20, sw_power_cap 0x4)."""
    sys.path.insert(0, ROOT)
    import bench

    s = bench.ClockSampler(0)
    s.t_begin = 10.0
    s.samples = [(9.0, 600.0, 1965.0, 200.0, 0x8),       # before the region: ignored
                 (10.5, 1400.0, 1965.0, 900.0, 0x4),
                 (11.0, 1500.0, 1965.0, 910.0, 0x0),
                 (11.5, 1600.0, 1965.0, 920.0, 0x4 | 0x20)]
    d = s.summary()
    assert d["samples"] == 3 and d["sm_mhz"] == 1500.0 and d["sm_max_mhz"] == 1965.0
    assert d["reasons"] == ["sw_power_cap", "sw_thermal_slowdown"]
    assert d["source"] == "nvml"
    empty = bench.ClockSampler(0)
    empty.t_begin = 0.0
    assert empty.summary()["samples"] == 0
