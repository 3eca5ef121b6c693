"""The bench.py JSON line keeps the driver's contract: checked on the committed round bench
line (profiles/r01_bench.json, produced by `python bench.py` on a B200) and on the
reference arm's line shape (CPU only)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line():
    with open(os.path.join(ROOT, "profiles", "r01_bench.json")) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_bench_line_has_the_contract_keys():
    d = _line()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["higher_is_better"] is True and d["scaling"] in ("weak", "strong")
    assert "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and 0.0 < r["frac"] <= 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("reference", "port")
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_value_is_the_metric_of_the_step_time():
    d = _line()
    n = d["config"]["n"]
    assert abs(d["value"] - 2.0 * n ** 3 / (d["ms_per_step"] * 1e-3) / 1e12) <= 1e-6 * d["value"]


def test_bench_gpus_n_without_n_devices_fails_loudly():
    """`bench.py --gpus N` outside torchrun re-launches itself as N ranks; with fewer than N
    visible GPUs (none here) it must exit non-zero instead of timing one GPU."""
    import subprocess
    import sys

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "--gpus 2" in r.stderr


def test_reference_arm_does_not_load_the_product_library():
    """The reference arm's process maps only oracle/ libraries (its inputs come from the
    oracle's restatement of the reference generator)."""
    import subprocess
    import sys

    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0',"
            "'--ref-n','64']; import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); print('PRODUCT_LOADED' if 'libipt_b200' in maps else 'CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "CLEAN" in r.stdout
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert line["impl"] == "reference" and line["config"]["reference_sample_n"] == 64
    assert line["config"]["same_config"] is False
