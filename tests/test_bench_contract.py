"""bench.py's JSON line contract (the driver parses it): the reference arm
runs anywhere (host only, no product library), the GPU arm on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, env=None, timeout=900):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout, env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_line_and_no_product_library():
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1',"
            " '--steps', '2', '--warmup', '3']; runpy.run_path('bench.py', run_name='__main__');"
            " print('MAPS', [l.split()[-1] for l in open('/proc/self/maps') if 'libpba' in l])")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = r.stdout.strip().splitlines()
    line = json.loads(lines[-2])
    assert lines[-1] == "MAPS []"  # the product library is never mapped
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference" and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] == 3
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the same config object as the GPU arm (bench.workload_config)
    assert line["config"]["pairs"] == 24 and line["config"]["pixel_pairs_per_iteration"] == 460800
    assert line["ms_per_step"] > 0 and line["value"] > 0


@pytest.mark.gpu
def test_gpu_arm_line():
    pytest.importorskip("torch")
    line = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-e2e-api"])
    assert BASE_KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["dtype"] == "f64"
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and 0 < roof["frac"] < 1.5 and roof["peak"] > 0
    assert line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["cpu_baseline"]["kind"] == "port"
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
    # c1 fits the device-resident LM loop: the timed steps are one conditional-graph launch
    assert line["parallelism"] == "single GPU, device-resident LM loop"
    host = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-e2e-api",
                 "--no-cpu-baseline", "--lm-loop", "host"])
    assert host["parallelism"] == "single GPU" and host["config"] == line["config"]
    ref = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3"])
    assert ref["config"] == line["config"]  # the driver compares them
